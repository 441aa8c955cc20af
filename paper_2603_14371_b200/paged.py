"""Unified paged KV pool: block allocator binding and cache handles.

One pool per backend holds every request's KV on HBM in fixed-size blocks
(SURVEY.md Appendix D).  A cache is a *handle* ``(pool, block_ids, seq_len)``:
the prefill writes blocks once, the action expert reads the same handle
(cross-task sharing, ``kvweaver/scheduler.py:112-120``), and language decode
extends it in place, copying a shared partially-filled tail block only when
another handle already wrote past it.  Handles keep the reference's value
semantics (``kvweaver/kv_manager.py:28-32``): an old handle still reads
exactly its positions after any later decode.

Block ids are assigned by the C++ allocator (``csrc/allocator.cpp``);
``oracle/paged_alloc.py`` restates the same rules and the CPU tests replay
random op sequences through both, comparing block tables, copy-on-write
triples and the full allocator state after every op (bit-exact).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .kv_manager import KvLayer

__all__ = ["BlockAllocator", "PagedKvCache"]


class BlockAllocator:
    """Owner of an ``oxy_alloc`` (block policy in C++) plus admission control.

    The reference checks capacity only when a request is stored and lets decode
    grow caches freely (``kvweaver/kv_manager.py:195-238``).  A physical pool
    must keep that promise: ``promise_budget`` sets aside, when a request is
    admitted, every block its decode can still take (ceil((P + max_len) / B)
    minus the prefix blocks, plus one copy-on-write copy of a shared tail), so
    a decode of admitted requests never runs out of blocks; allocations that
    are not covered by a promise (prefills, forks of a state) only use blocks
    nobody was promised, and fail loudly (``MemoryError``) up front instead."""

    def __init__(self, num_blocks: int, block_size: int):
        self.num_blocks = int(num_blocks)
        self.block_size = int(block_size)
        self.promised = 0
        h = C.c_void_p()
        _lib.call("oxy_alloc_create", C.c_int32(num_blocks), C.c_int32(block_size), C.byref(h))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().oxy_alloc_destroy(h)
            except Exception:
                pass
            self._h = None

    def blocks_for(self, n: int) -> int:
        return -(-n // self.block_size)

    def unpromised_free(self) -> int:
        return self.num_free - self.promised

    def promise_budget(self, kv, max_len: int) -> None:
        """Admission: set aside the blocks ``kv``'s request can take while decoding
        up to ``max_len`` tokens; the promise travels with the handle through decodes."""
        n = self.blocks_for(kv.seq_len + max_len) - self.blocks_for(kv.seq_len) + 1
        if n > self.unpromised_free():
            raise MemoryError(f"KV pool capacity exceeded: admitting a request needs {n} blocks, "
                              f"{self.unpromised_free()} free and not promised to live requests")
        self.promised += n
        kv.promise += n

    def alloc_seq(self, n_tokens: int) -> tuple[int, ...]:
        if self.blocks_for(n_tokens) > self.unpromised_free():
            raise MemoryError(f"KV pool out of blocks: a {n_tokens}-position prefix needs "
                              f"{self.blocks_for(n_tokens)}, {self.unpromised_free()} free and not "
                              f"promised to live requests")
        out = np.empty(self.blocks_for(n_tokens), np.int32)
        _lib.call("oxy_alloc_seq", self._h, C.c_int32(n_tokens), _lib.ptr_i32(out))
        return tuple(out.tolist())

    def incref(self, blocks) -> None:
        b = _lib.as_i32(blocks)
        _lib.call("oxy_alloc_incref", self._h, _lib.ptr_i32(b), C.c_int32(len(b)))

    def decref(self, blocks) -> None:
        if self._h is None or not self._h.value:  # allocator already torn down (GC order)
            return
        b = _lib.as_i32(blocks)
        _lib.call("oxy_alloc_decref", self._h, _lib.ptr_i32(b), C.c_int32(len(b)))

    def reserve(self, blocks, seq_len: int, n_new: int):
        b = _lib.as_i32(blocks)
        out = np.empty(self.blocks_for(seq_len + n_new), np.int32)
        cow = np.empty(3, np.int32)
        _lib.call("oxy_alloc_reserve", self._h, _lib.ptr_i32(b), C.c_int32(seq_len),
                  C.c_int32(n_new), _lib.ptr_i32(out), _lib.ptr_i32(cow))
        return out, cow

    def settle(self, blocks: np.ndarray, seq_len: int, n_reserved: int, n_actual: int):
        nb = C.c_int32()
        _lib.call("oxy_alloc_settle", self._h, _lib.ptr_i32(blocks), C.c_int32(seq_len),
                  C.c_int32(n_reserved), C.c_int32(n_actual), C.byref(nb))
        return tuple(blocks[:nb.value].tolist())

    @property
    def num_free(self) -> int:
        n = C.c_int32()
        _lib.call("oxy_alloc_num_free", self._h, C.byref(n))
        return n.value

    def snapshot(self):
        ref = np.empty(self.num_blocks, np.int32)
        fill = np.empty(self.num_blocks, np.int32)
        free = np.empty(self.num_blocks, np.int32)
        n = C.c_int32()
        _lib.call("oxy_alloc_snapshot", self._h, _lib.ptr_i32(ref), _lib.ptr_i32(fill),
                  _lib.ptr_i32(free), C.byref(n))
        return ref, fill, free[:n.value].copy()

    def reserve_need(self, kv, n_new: int) -> int:
        b = _lib.as_i32(kv.blocks)
        need = C.c_int32()
        _lib.call("oxy_alloc_reserve_need", self._h, _lib.ptr_i32(b), C.c_int32(kv.seq_len),
                  C.c_int32(n_new), C.byref(need))
        return need.value

    def reserve_rows(self, caches, n_new):
        """``reserve`` for every row of a decode batch.  A row draws first on its
        handle's promise (the first row of a handle; forks of one state draw on
        the unpromised free blocks only); a row needing more than that plus the
        unpromised free blocks fails up front (``MemoryError``).  On any failure
        the rows already reserved are rolled back — blocks, copy-on-write copies
        and raised tail watermarks — so a failed call leaves the allocator as it
        found it.  Returns the tables, copy-on-write triples and the promised
        blocks each row drew on (``carry_promises`` settles them after the call)."""
        tables, cows, drawn = [], [], []
        seen, pending = set(), 0  # handles whose promise is taken; promised blocks drawn so far
        try:
            for kv, n in zip(caches, n_new):
                need = self.reserve_need(kv, n)
                own = kv.promise if id(kv) not in seen else 0
                seen.add(id(kv))
                use = min(own, need)
                spare = self.num_free - (self.promised - pending)
                if need - use > spare:
                    raise MemoryError(f"KV pool out of blocks: a decode row needs {need} blocks, "
                                      f"{use} of them admitted, {spare} free and not promised")
                t, c = self.reserve(kv.blocks, kv.seq_len, n)
                pending += use
                tables.append(t)
                cows.append(c)
                drawn.append(use)
        except BaseException:
            self.unreserve(tables, [kv.seq_len for kv in caches], n_new)
            raise
        return tables, cows, drawn

    def carry_promises(self, olds, news, drawn) -> None:
        """After a decode: the blocks a row kept (new tail blocks, a copy-on-write
        copy) come out of its promise; the rest of the promise moves to the row's
        new handle."""
        for old, new, d in zip(olds, news, drawn):
            n_old = len(old.blocks)
            kept = len(new.blocks) - n_old + (1 if new.blocks[n_old - 1] != old.blocks[-1] else 0)
            use = min(d, max(0, kept))
            self.promised -= use
            new.promise += old.promise - use
            old.promise = 0

    def unreserve(self, tables, seq_lens, n_new) -> None:
        """Undo ``reserve`` for rows that wrote nothing: settle at zero new
        positions (frees fresh blocks, restores the tail watermark), then drop
        the references the reservation took."""
        for t, s, n in zip(tables, seq_lens, n_new):
            self.decref(self.settle(t, s, n, 0))

    def slot_mapping(self, blocks, start: int, count: int) -> np.ndarray:
        b = _lib.as_i32(blocks)
        out = np.empty(count, np.int32)
        _lib.call("oxy_build_slot_mapping", _lib.ptr_i32(b), C.c_int32(self.block_size),
                  C.c_int32(start), C.c_int32(count), _lib.ptr_i32(out))
        return out


class PagedKvCache:
    """Cache handle into a backend's pool.  Duck-types ``KvCache``:
    ``seq_len``, ``backend_tag``, ``num_layers``, ``layers`` (materialised
    lazily from HBM as read-only float64 ``KvLayer``s) and value equality.
    Dropping the last reference returns the blocks to the pool."""

    __slots__ = ("owner", "blocks", "seq_len", "backend_tag", "promise", "__weakref__")

    def __init__(self, owner, blocks: tuple, seq_len: int):
        self.owner = owner
        self.blocks = tuple(blocks)
        self.seq_len = int(seq_len)
        self.backend_tag = owner.backend_tag
        self.promise = 0  # blocks set aside for this handle's request (BlockAllocator.promise_budget)

    def share(self) -> "PagedKvCache":
        """A second handle on the same blocks (refcounted): one per request when
        several language tasks start from one observation's prefix."""
        self.owner.allocator.incref(self.blocks)
        return PagedKvCache(self.owner, self.blocks, self.seq_len)

    def __del__(self):
        owner = getattr(self, "owner", None)
        if owner is not None and self.blocks:
            try:
                owner.allocator.promised -= self.promise  # the request is gone
                owner.allocator.decref(self.blocks)
            except Exception:
                pass

    @property
    def num_layers(self) -> int:
        return self.owner.num_layers

    @property
    def layers(self) -> tuple:
        """Read from HBM on every access (no host memo): a check such as the
        sharing suite's "denoise left the cache untouched"
        (``kvweaver/verify.py:241-247``) must see the pool, not a stale copy."""
        return tuple(KvLayer(*self.owner.read_kv(self, l)) for l in range(self.num_layers))

    def __eq__(self, other):
        if not hasattr(other, "backend_tag") or not hasattr(other, "layers"):
            return NotImplemented
        if self.backend_tag != other.backend_tag or self.seq_len != other.seq_len:
            return False
        if isinstance(other, PagedKvCache) and other.owner is self.owner \
                and other.blocks == self.blocks:
            return True
        return self.layers == tuple(other.layers)

    __hash__ = None

    def __repr__(self):
        return f"PagedKvCache(seq_len={self.seq_len}, blocks={self.blocks})"
