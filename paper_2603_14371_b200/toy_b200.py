"""F1 backend: the reference toy transformer computed on the B200.

Drop-in for ``kvweaver.ToyBackend`` (``kvweaver/backend.py:235-420``): same
constructor, same three operations, same validation messages, same
``recompute_logits`` oracle route and the private weight hooks the reference
tests poke (``_embed``, ``_unembed``, ``_action_head``).  The math runs in
``csrc/toy.cu`` in fp32 verification mode (or fp64), the KV lives in the
unified paged pool, and the k-step decode loop with per-row termination runs
on the device with one host round trip per call.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .backend import ActionChunk, BackendConfig, CostModelParams, Observation, PricedBackend
from .kv_manager import BatchedState
from .paged import BlockAllocator, PagedKvCache

__all__ = ["ToyBackend"]

_DTYPES = {"f32": 0, "f64": 1}
_WEIGHTS = {"_embed": 0, "_unembed": 7, "_action_head": 8}
_BIG_BUDGET = 1 << 30


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 backends need a CUDA device (no CPU fallback)")
    _lib.lib()


class ToyBackend(PricedBackend):
    def __init__(self, config: BackendConfig | None = None, cost: CostModelParams | None = None,
                 dtype: str = "f32", num_blocks: int = 4096, block_size: int = 16):
        require_cuda()
        self.config = c = config or BackendConfig()
        self.cost = cost or CostModelParams.zero()
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}, got {dtype!r}")
        self.dtype = dtype
        self.backend_tag = f"toy/L{c.L}-d{c.d_model}-h{c.n_heads}-v{c.vocab}-s{c.seed}/b200-{dtype}"
        self.kind = "Toy"
        self.num_layers = c.L
        self.block_size = block_size
        self.allocator = BlockAllocator(num_blocks, block_size)
        cfg = _lib.OxyToyConfig(c.L, c.d_model, c.n_heads, c.vocab, c.eos_token, c.action_dim,
                                c.H, c.seed & ((1 << 64) - 1))
        h = C.c_void_p()
        _lib.call("oxy_toy_create", C.byref(cfg), C.c_int32(_DTYPES[dtype]),
                  C.c_int32(num_blocks), C.c_int32(block_size), _lib.stream_ptr(), C.byref(h))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().oxy_toy_destroy(h)
            except Exception:
                pass
            self._h = None

    # ------------------------------------------------------------ weights

    def _weight(self, which: int, layer: int = 0, value=None) -> np.ndarray:
        c = self.config
        shapes = {0: (c.vocab, c.d_model), 7: (c.d_model, c.vocab),
                  8: (c.H * c.action_dim, c.d_model)}
        shape = shapes[which]
        if value is None:
            out = np.empty(shape, np.float64)
            _lib.call("oxy_toy_weight", self._h, C.c_int32(which), C.c_int32(layer),
                      _lib.ptr_f64(out), C.c_int64(out.size), C.c_int32(0), _lib.stream_ptr())
            out.flags.writeable = False
            return out
        buf = np.ascontiguousarray(value, dtype=np.float64)
        if buf.shape != shape:
            raise ValueError(f"weight shape {buf.shape} != {shape}")
        _lib.call("oxy_toy_weight", self._h, C.c_int32(which), C.c_int32(layer),
                  _lib.ptr_f64(buf), C.c_int64(buf.size), C.c_int32(1), _lib.stream_ptr())
        return buf

    def __getattr__(self, name):
        if name in _WEIGHTS:
            return self._weight(_WEIGHTS[name])
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in _WEIGHTS:
            self._weight(_WEIGHTS[name], value=value)
        else:
            object.__setattr__(self, name, value)

    # ------------------------------------------------------------ pool access

    def read_kv(self, kv: PagedKvCache, layer: int):
        d = self.config.d_model
        keys = np.empty((kv.seq_len, d), np.float64)
        vals = np.empty((kv.seq_len, d), np.float64)
        b = _lib.as_i32(kv.blocks)
        _lib.call("oxy_toy_read_kv", self._h, _lib.ptr_i32(b), C.c_int32(kv.seq_len),
                  C.c_int32(layer), _lib.ptr_f64(keys), _lib.ptr_f64(vals), _lib.stream_ptr())
        return keys, vals

    def write_kv(self, kv: PagedKvCache, layer: int, keys, values) -> None:
        """Overwrite one layer's rows of a handle (inverse of ``read_kv``)."""
        d = self.config.d_model
        k = np.ascontiguousarray(keys, np.float64).reshape(kv.seq_len, d)
        v = np.ascontiguousarray(values, np.float64).reshape(kv.seq_len, d)
        b = _lib.as_i32(kv.blocks)
        _lib.call("oxy_toy_write_kv", self._h, _lib.ptr_i32(b), C.c_int32(kv.seq_len),
                  C.c_int32(layer), _lib.ptr_f64(k), _lib.ptr_f64(v), _lib.stream_ptr())

    def adopt(self, kv) -> PagedKvCache:
        """Copy a host ``KvCache`` (e.g. one produced by the reference package)
        into this backend's pool and return the resident handle."""
        if kv.num_layers != self.num_layers:
            raise ValueError(f"cache has {kv.num_layers} layers, backend has {self.num_layers}")
        h = PagedKvCache(self, self.allocator.alloc_seq(kv.seq_len), kv.seq_len)
        for l, layer in enumerate(kv.layers):
            self.write_kv(h, l, layer.keys, layer.values)
        return h

    def _own(self, kv) -> PagedKvCache:
        """The pool-resident handle for ``kv``.  A cache of the same backend tag that
        lives elsewhere (a host ``KvCache`` — e.g. one a caller rebuilt from
        ``layers`` — or another instance's pool) is accepted as the reference accepts
        any cache with a matching tag (``kvweaver/backend.py:179-183``): its layers
        are copied into this pool (``adopt``)."""
        self._check_tag(kv)
        if isinstance(kv, PagedKvCache) and kv.owner is self:
            return kv
        if hasattr(kv, "layers") and hasattr(kv, "seq_len"):
            return self.adopt(kv)
        raise ValueError(f"cache from backend {kv.backend_tag!r} is not resident in this "
                         f"backend's KV pool")

    # ------------------------------------------------------------ protocol

    def recompute_logits(self, token_ids) -> np.ndarray:
        toks = _lib.as_i32(list(token_ids))
        out = np.empty(self.config.vocab, np.float64)
        _lib.call("oxy_toy_recompute_logits", self._h, _lib.ptr_i32(toks), C.c_int32(len(toks)),
                  _lib.ptr_f64(out), _lib.stream_ptr())
        return out

    def prefill(self, obs: Observation) -> PagedKvCache:
        self._check_obs(obs)
        toks = _lib.as_i32(obs.obs_tokens)
        blocks = self.allocator.alloc_seq(len(toks))
        kv = PagedKvCache(self, blocks, len(toks))   # owns the blocks from here on
        b = _lib.as_i32(blocks)
        _lib.call("oxy_toy_prefill", self._h, _lib.ptr_i32(toks), C.c_int32(len(toks)),
                  _lib.ptr_i32(b), _lib.stream_ptr())
        return kv

    def action_denoise(self, kv, S: int) -> ActionChunk:
        self._check_tag(kv)
        if S < 1:
            raise ValueError(f"denoise step count must be >= 1, got {S}")
        kv = self._own(kv)
        c = self.config
        out = np.empty(c.H * c.action_dim, np.float64)
        b = _lib.as_i32(kv.blocks)
        _lib.call("oxy_toy_denoise", self._h, _lib.ptr_i32(b), C.c_int32(kv.seq_len),
                  C.c_int32(S), _lib.ptr_f64(out), _lib.stream_ptr())
        return ActionChunk(out.reshape(c.H, c.action_dim))

    def batched_language_decode(self, batched: BatchedState, k: int) -> BatchedState:
        self._check_batch(batched, k)
        c = self.config
        m = batched.size
        caches = [self._own(kv) for kv in batched.kv_batch]
        budgets, reserved, lasts = [], [], []
        for toks, max_len in zip(batched.token_buffers, batched.max_lens):
            left = max_len - len(toks)
            budgets.append(left if left > 0 else _BIG_BUDGET)
            reserved.append(min(k, left) if left > 0 else k)
            lasts.append(toks[-1] if toks else c.eos_token)
        tables, cows, drawn = self.allocator.reserve_rows(caches, reserved)
        maxb = max(len(t) for t in tables)
        bt = np.zeros((m, maxb), np.int32)
        for i, t in enumerate(tables):
            bt[i, :len(t)] = t
        seq = _lib.as_i32([kv.seq_len for kv in caches])
        last = _lib.as_i32(lasts)
        bud = _lib.as_i32(budgets)
        cow = _lib.as_i32(np.stack(cows))
        out = np.empty((m, k), np.int32)
        cnt = np.empty(m, np.int32)
        try:
            _lib.call("oxy_toy_decode", self._h, C.c_int32(m), C.c_int32(k), _lib.ptr_i32(bt),
                      C.c_int32(maxb), _lib.ptr_i32(seq), _lib.ptr_i32(last), _lib.ptr_i32(bud),
                      _lib.ptr_i32(cow), _lib.ptr_i32(out), _lib.ptr_i32(cnt), _lib.stream_ptr())
        except BaseException:
            self.allocator.unreserve(tables, [kv.seq_len for kv in caches], reserved)
            raise
        new_caches, bufs, flags = [], [], []
        for i, kv in enumerate(caches):
            adv = int(cnt[i])
            blocks = self.allocator.settle(tables[i], kv.seq_len, reserved[i], adv)
            new_caches.append(PagedKvCache(self, blocks, kv.seq_len + adv))
            toks = batched.token_buffers[i] + tuple(int(t) for t in out[i, :adv])
            bufs.append(toks)
            flags.append(bool(adv and (toks[-1] == c.eos_token or len(toks) == batched.max_lens[i])))
        self.allocator.carry_promises(caches, new_caches, drawn)
        return BatchedState(tuple(new_caches), tuple(bufs), tuple(flags), batched.request_ids,
                            batched.max_lens, batched.created_frames)
