"""F2 backend: a pi0.5-shaped Mixture-of-Transformers VLA on the B200.

Same protocol as the reference backends (``kvweaver/backend.py:163-201``):
``prefill`` writes the shared observation prefix (3 SigLIP cameras + prompt)
into the unified paged KV pool ONCE; ``action_denoise`` runs the
flow-matching action expert whose suffix attends to that same paged prefix
(cross-task KV sharing, ``PAPER.md:217-238``); ``batched_language_decode``
continues language requests from the same handles, continuously batched
across frames.  ``admit_many`` batches the prefill and denoise of r
lock-stepped robot streams (``Uniform(r)`` arrivals).

Shapes (``Pi05Config``) follow the public openpi pi0.5 configuration
(SURVEY.md Appendix B); weights are random (splitmix64 counter draws,
U(+-sqrt(3/fan_in))), which the reference cannot pin: this family's layer
arithmetic is checked against ``oracle/pi05_ref.py`` (torch fp32), parity
unpinned by the reference itself.  Compute is bf16 on tcgen05 with fp32
accumulation and an fp32 residual stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .backend import ActionChunk, CostModelParams, Observation, PricedBackend
from .kv_manager import BatchedState, GenerationState, KvLayer
from .paged import BlockAllocator, PagedKvCache
from .timing import StageMeter

__all__ = ["Pi05Config", "Pi05Observation", "Pi05Backend", "TINY", "synthetic_images"]

KV_BLOCK = 64
HEAD_DIM = 256
_BIG_BUDGET = 1 << 30


class OxyPi05Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "width", "depth", "mlp", "vocab", "expert_width", "expert_mlp", "vit_width", "vit_depth",
        "vit_mlp", "vit_heads", "H", "action_dim", "eos_token")] + [("seed", C.c_uint64)]


@dataclass(frozen=True, slots=True)
class Pi05Config:
    """pi0.5 shape.  Defaults: Gemma-2B + Gemma-300M expert + SigLIP So400m/14."""

    width: int = 2048
    depth: int = 18
    mlp: int = 16384
    vocab: int = 257152
    expert_width: int = 1024
    expert_mlp: int = 4096
    vit_width: int = 1152
    vit_depth: int = 27
    vit_mlp: int = 4304
    vit_heads: int = 16
    H: int = 50
    action_dim: int = 32
    S: int = 10
    eos_token: int = 1
    seed: int = 7
    n_cams: int = 3

    def __post_init__(self):
        for name in ("width", "expert_width", "mlp", "expert_mlp"):
            if getattr(self, name) % 64:
                raise ValueError(f"{name} must be a multiple of 64")
        if self.vit_depth and self.vit_width != 72 * self.vit_heads:
            raise ValueError("vision head dim must be 72 (vit_width = 72 * vit_heads)")
        if not 0 <= self.eos_token < self.vocab:
            raise ValueError(f"eos_token {self.eos_token} outside vocab of {self.vocab}")
        if self.H < 1 or self.S < 1 or self.action_dim < 1:
            raise ValueError("action_dim, H and S must be positive")

    @property
    def L(self) -> int:
        return self.depth

    def to_c(self) -> OxyPi05Config:
        return OxyPi05Config(self.width, self.depth, self.mlp, self.vocab, self.expert_width,
                             self.expert_mlp, self.vit_width, self.vit_depth, self.vit_mlp,
                             self.vit_heads, self.H, self.action_dim, self.eos_token,
                             self.seed & ((1 << 64) - 1))


# reduced shape with the same code paths (parity tests against the CPU oracle)
TINY = Pi05Config(width=256, depth=2, mlp=512, vocab=1000, expert_width=128, expert_mlp=256,
                  vit_width=144, vit_depth=2, vit_mlp=288, vit_heads=2, H=10, action_dim=8,
                  S=4, eos_token=1, seed=3, n_cams=2)


@dataclass(frozen=True, slots=True, eq=False)
class Pi05Observation:
    """Observation with camera images: uint8 [n_cams, 224, 224, 3] on host
    (numpy) or device (torch CUDA tensor), plus prompt token ids."""

    obs_tokens: tuple
    frame: int
    images: object = None

    def __post_init__(self):
        object.__setattr__(self, "obs_tokens", tuple(self.obs_tokens))
        n = 0 if self.images is None else int(self.images.shape[0])
        if n == 0 and not self.obs_tokens:
            raise ValueError("observation needs at least one token")
        if n and tuple(self.images.shape[1:]) != (224, 224, 3):
            raise ValueError(f"images must be [n, 224, 224, 3], got {tuple(self.images.shape)}")

    @property
    def n_images(self) -> int:
        return 0 if self.images is None else int(self.images.shape[0])

    @property
    def prefix_len(self) -> int:
        return 256 * self.n_images + len(self.obs_tokens)


def _as_pi05(cfg) -> Pi05Config:
    if cfg is None:
        return Pi05Config()
    if isinstance(cfg, Pi05Config):
        return cfg
    # a reference BackendConfig: keep the protocol fields, pi0.5 shape otherwise
    return Pi05Config(H=cfg.H, S=cfg.S, action_dim=cfg.action_dim, seed=cfg.seed,
                      vocab=max(cfg.vocab, 2), eos_token=cfg.eos_token, width=256, depth=2,
                      mlp=512, expert_width=128, expert_mlp=256, vit_depth=0)


class DeferredActionChunk(ActionChunk):
    """An ActionChunk whose values are still being copied to the host behind a CUDA
    event: the first read of ``actions`` waits for the event and converts and
    validates exactly as ``ActionChunk`` does (same float64 values, same errors).
    Returned by an overlapped frame's join when no stage meter is attached, so the
    frame call returns without waiting for its denoise and the host enqueues the
    next frame while the action expert is still running."""

    __slots__ = ("_host", "_row", "_done", "_val")

    def __init__(self, host, row: int, done):
        object.__setattr__(self, "_host", host)  # pinned torch tensor [n, H, A] (kept alive)
        object.__setattr__(self, "_row", row)
        object.__setattr__(self, "_done", done)
        object.__setattr__(self, "_val", None)

    @property
    def actions(self) -> np.ndarray:
        v = self._val
        if v is None:
            self._done.synchronize()
            v = ActionChunk(self._host[self._row].numpy().astype(np.float64)).actions
            object.__setattr__(self, "_val", v)
        return v

    def __repr__(self) -> str:
        return f"DeferredActionChunk(actions={self.actions!r})"


class Pi05Backend(PricedBackend):
    def __init__(self, config=None, cost: CostModelParams | None = None, num_blocks: int = 2048,
                 measure: bool = False, overlap: bool = True):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("Pi05Backend needs a CUDA device (no CPU fallback)")
        self.config = c = _as_pi05(config)
        self.cost = cost or CostModelParams.zero()
        self.kind = "Pi05"
        self.backend_tag = (f"pi05/w{c.width}-d{c.depth}-e{c.expert_width}-v{c.vocab}"
                            f"-vit{c.vit_depth}-s{c.seed}")
        self.num_layers = c.depth
        self.block_size = KV_BLOCK
        self.allocator = BlockAllocator(num_blocks, KV_BLOCK)
        self.meter = StageMeter() if measure else None
        self._stage = [(None, None), (None, None)]  # pinned image staging ring (host frames)
        self._stage_next = 0
        if not overlap:   # stage-serial frames (the reference's order, scheduler.py:117-171)
            self.admit_overlapped = None
        h = C.c_void_p()
        _lib.call("oxy_pi05_create", C.byref(c.to_c()), C.c_int32(num_blocks), _lib.stream_ptr(),
                  C.byref(h))
        self._h = h
        self._torch = torch

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().oxy_pi05_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---------------------------------------------------------------- utils

    def _span(self, stage):
        import contextlib
        return self.meter.span(stage) if self.meter is not None else contextlib.nullcontext()

    def tensors(self) -> list[dict]:
        n = C.c_int32()
        _lib.call("oxy_pi05_num_tensors", self._h, C.byref(n))
        out = []
        for i in range(n.value):
            name = C.create_string_buffer(64)
            shape = (C.c_int64 * 2)()
            dt, off = C.c_int32(), C.c_uint64()
            bound, center = C.c_float(), C.c_float()
            _lib.call("oxy_pi05_tensor_info", self._h, C.c_int32(i), name, shape, C.byref(dt),
                      C.byref(off), C.byref(bound), C.byref(center))
            out.append(dict(index=i, name=name.value.decode(), shape=(shape[0], shape[1]),
                            dtype="bf16" if dt.value == 0 else "f32", offset=off.value,
                            bound=bound.value, center=center.value))
        return out

    def read_tensor(self, info: dict):
        """Weight tensor as a torch CPU tensor (bf16 or f32)."""
        torch = self._torch
        dtype = torch.bfloat16 if info["dtype"] == "bf16" else torch.float32
        t = torch.empty(info["shape"], dtype=dtype)
        _lib.call("oxy_pi05_tensor_read", self._h, C.c_int32(info["index"]),
                  C.c_void_p(t.data_ptr()), C.c_int64(t.numel() * t.element_size()),
                  _lib.stream_ptr())
        return t

    def read_kv(self, kv: PagedKvCache, layer: int):
        keys = np.empty((kv.seq_len, HEAD_DIM), np.float32)
        vals = np.empty((kv.seq_len, HEAD_DIM), np.float32)
        b = _lib.as_i32(kv.blocks)
        _lib.call("oxy_pi05_read_kv", self._h, _lib.ptr_i32(b), C.c_int32(kv.seq_len),
                  C.c_int32(layer), keys.ctypes.data_as(C.c_void_p),
                  vals.ctypes.data_as(C.c_void_p), _lib.stream_ptr())
        return keys.astype(np.float64), vals.astype(np.float64)

    def _own(self, kv) -> PagedKvCache:
        self._check_tag(kv)
        if not isinstance(kv, PagedKvCache) or kv.owner is not self:
            raise ValueError(f"cache from backend {kv.backend_tag!r} is not resident in this "
                             f"backend's KV pool")
        return kv

    def _check_obs(self, obs) -> None:
        v = self.config.vocab
        for t in obs.obs_tokens:
            if not 0 <= t < v:
                raise ValueError(f"observation token {t} outside vocab of {v}")

    def _images_device(self, obs_list):
        torch = self._torch
        imgs = [o.images for o in obs_list if getattr(o, "images", None) is not None
                and o.images.shape[0] > 0]
        if not imgs:
            return None, None
        if all(isinstance(i, torch.Tensor) and i.is_cuda for i in imgs):
            dev = imgs[0] if len(imgs) == 1 else torch.cat(imgs)
        else:
            parts = [np.asarray(i.cpu() if isinstance(i, torch.Tensor) else i, dtype=np.uint8) for i in imgs]
            nbytes = sum(p.nbytes for p in parts)
            # one copy into a reused pinned staging buffer (a ring of two; the H2D copy
            # that last read a slot is waited for before it is overwritten), then an
            # asynchronous H2D on the caller's stream
            slot = self._stage_next
            self._stage_next ^= 1
            buf, ev = self._stage[slot]
            if buf is None or buf.numel() < nbytes:
                buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
            elif ev is not None:
                ev.synchronize()
            flat = buf.numpy()
            off = 0
            for p in parts:
                flat[off:off + p.nbytes] = p.reshape(-1)
                off += p.nbytes
            shape = (sum(p.shape[0] for p in parts),) + parts[0].shape[1:]
            dev = buf[:nbytes].to("cuda", non_blocking=True).view(shape)
            ev = torch.cuda.Event()
            ev.record()
            self._stage[slot] = (buf, ev)
        return dev.contiguous(), C.c_void_p(dev.data_ptr())

    # ---------------------------------------------------------------- protocol

    def prefill_many(self, obs_list) -> list[PagedKvCache]:
        for o in obs_list:
            self._check_obs(o)
        n_img = _lib.as_i32([getattr(o, "n_images", 0) for o in obs_list])
        n_txt = _lib.as_i32([len(o.obs_tokens) for o in obs_list])
        toks = _lib.as_i32([t for o in obs_list for t in o.obs_tokens] or [0])
        handles = []
        for o, ni, nt in zip(obs_list, n_img, n_txt):
            p = 256 * int(ni) + int(nt)
            handles.append(PagedKvCache(self, self.allocator.alloc_seq(p), p))
        blocks = _lib.as_i32([b for h in handles for b in h.blocks])
        with self._span("prefill"):
            keep, img_ptr = self._images_device(obs_list)
            _lib.call("oxy_pi05_prefill", self._h, C.c_int32(len(obs_list)), _lib.ptr_i32(n_img),
                      _lib.ptr_i32(n_txt), _lib.ptr_i32(toks), img_ptr, _lib.ptr_i32(blocks),
                      _lib.stream_ptr())
        del keep
        return handles

    def prefill(self, obs) -> PagedKvCache:
        return self.prefill_many([obs])[0]

    def denoise_many(self, kvs, S: int) -> list[ActionChunk]:
        if S < 1:
            raise ValueError(f"denoise step count must be >= 1, got {S}")
        kvs = [self._own(kv) for kv in kvs]
        c = self.config
        torch = self._torch
        out = torch.empty((len(kvs), c.H, c.action_dim), dtype=torch.float32, device="cuda")
        lens = _lib.as_i32([kv.seq_len for kv in kvs])
        blocks = _lib.as_i32([b for kv in kvs for b in kv.blocks])
        with self._span("denoise"):
            _lib.call("oxy_pi05_denoise", self._h, C.c_int32(len(kvs)), _lib.ptr_i32(lens),
                      _lib.ptr_i32(blocks), C.c_int32(S), C.c_void_p(out.data_ptr()),
                      _lib.stream_ptr())
            host = out.cpu().numpy().astype(np.float64)
        return [ActionChunk(a) for a in host]

    def action_denoise(self, kv, S: int) -> ActionChunk:
        self._check_tag(kv)
        return self.denoise_many([kv], S)[0]

    def admit_many(self, arrivals, t: int):
        """Lock-stepped streams: one batched prefill and one batched denoise."""
        kvs = self.prefill_many([a.observation for a in arrivals])
        chunks = self.denoise_many(kvs, self.config.S)
        return [(chunk, GenerationState(kv, (), False, t, a.n_tokens))
                for chunk, kv, a in zip(chunks, kvs, arrivals)]

    def admit_overlapped(self, arrivals, t: int):
        """Prefill now; denoise on the model's action-expert lane without
        blocking the backend stream, so the frame's batched decode (enqueued
        next) runs concurrently with it.  Returns ``(states, join)``:
        ``join()`` orders the backend stream after the denoise and starts the
        action copy-out; the callable it returns yields the ActionChunks.
        """
        kvs = self.prefill_many([a.observation for a in arrivals])
        c = self.config
        torch = self._torch
        n = len(kvs)
        out = torch.empty((n, c.H, c.action_dim), dtype=torch.float32, device="cuda")
        lens = _lib.as_i32([kv.seq_len for kv in kvs])
        blocks = _lib.as_i32([b for kv in kvs for b in kv.blocks])
        _lib.call("oxy_pi05_denoise_async", self._h, C.c_int32(n), _lib.ptr_i32(lens),
                  _lib.ptr_i32(blocks), C.c_int32(c.S), C.c_void_p(out.data_ptr()),
                  _lib.stream_ptr())
        states = [GenerationState(kv, (), False, t, a.n_tokens) for kv, a in zip(kvs, arrivals)]

        def join():
            _lib.call("oxy_pi05_join", self._h, _lib.stream_ptr())
            host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
            host.copy_(out, non_blocking=True)
            done = torch.cuda.Event()
            done.record()

            def chunks():
                if self.meter is None:
                    return [DeferredActionChunk(host, i, done) for i in range(n)]
                done.synchronize()
                if self.meter is not None:
                    us = C.c_double()
                    _lib.call("oxy_pi05_denoise_elapsed_us", self._h, C.byref(us))
                    self.meter.put("denoise", us.value)
                return [ActionChunk(a) for a in host.numpy().astype(np.float64)]
            return chunks
        return states, join

    def recompute_logits(self, token_ids) -> np.ndarray:
        """No-cache logits of the last position (``kvweaver/backend.py:301-304``), the
        route ``suite_reference`` grades cached decode against: one dense forward over
        the whole sequence with a plain fp32 attention kernel — no pool, no block
        tables, no decode kernels.  The prefix (bidirectional, prefix-LM) is everything
        before the LAST EOS: the first decode input is EOS at position P
        (``kvweaver/backend.py:359-362``) and decoded tokens never contain EOS (a
        request stops on it), so the last EOS is that marker.  Without an EOS the
        whole sequence is prefix."""
        toks = _lib.as_i32([int(t) for t in token_ids])
        if len(toks) == 0:
            raise ValueError("recompute needs at least one token")
        v = self.config.vocab
        for t in toks:
            if not 0 <= t < v:
                raise ValueError(f"token {int(t)} outside vocab of {v}")
        eos = np.flatnonzero(toks == self.config.eos_token)
        p = int(eos[-1]) if len(eos) else len(toks)
        out = np.empty(v, np.float32)
        _lib.call("oxy_pi05_recompute_logits", self._h, _lib.ptr_i32(toks), C.c_int32(len(toks)),
                  C.c_int32(p), out.ctypes.data_as(C.c_void_p), _lib.stream_ptr())
        return out.astype(np.float64)

    def batched_language_decode(self, batched: BatchedState, k: int,
                                return_logits: bool = False):
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
        for i, tb in enumerate(tables):
            bt[i, :len(tb)] = tb
        seq = _lib.as_i32([kv.seq_len for kv in caches])
        out = np.empty((m, k), np.int32)
        cnt = np.empty(m, np.int32)
        logits = np.empty((k, m, c.vocab), np.float32) if return_logits else None
        try:
            with self._span("decode"):
                _lib.call("oxy_pi05_decode", self._h, C.c_int32(m), C.c_int32(k),
                          _lib.ptr_i32(bt), C.c_int32(maxb), _lib.ptr_i32(seq),
                          _lib.ptr_i32(_lib.as_i32(lasts)), _lib.ptr_i32(_lib.as_i32(budgets)),
                          _lib.ptr_i32(_lib.as_i32(np.stack(cows))), _lib.ptr_i32(out),
                          _lib.ptr_i32(cnt),
                          logits.ctypes.data_as(C.c_void_p) if return_logits else None,
                          _lib.stream_ptr())
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
            flags.append(bool(adv and (toks[-1] == c.eos_token
                                       or len(toks) == batched.max_lens[i])))
        self.allocator.carry_promises(caches, new_caches, drawn)
        res = BatchedState(tuple(new_caches), tuple(bufs), tuple(flags), batched.request_ids,
                           batched.max_lens, batched.created_frames)
        return (res, logits) if return_logits else res


def synthetic_images(n: int, seed: int) -> np.ndarray:
    """uint8 camera frames from a splitmix64 counter."""
    from .rng import counter_u64
    raw = counter_u64(seed, 0, n * 224 * 224 * 3 // 8 + 1).view(np.uint8)
    return raw[: n * 224 * 224 * 3].reshape(n, 224, 224, 3).copy()
