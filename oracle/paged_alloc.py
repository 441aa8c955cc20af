"""ORACLE — test infrastructure only; never imported by the product path.

Plain-Python restatement of the paged-KV block allocator implemented in
``paper_2603_14371_b200/csrc/allocator.cpp``.  The reference has no pool (its
caches are per-request numpy copies, ``kvweaver/kv_manager.py:35-105``); the
allocator rules are the builder's design pinned in SURVEY.md Appendix D and
DESIGN.md §3.  Tests replay random op sequences through both and require
bit-exact block tables, copy-on-write triples and allocator state.

Rules:
  * free blocks: min-heap, lowest id first;
  * refcount + fill watermark (slots claimed) per block;
  * alloc_seq(n): ceil(n/B) fresh blocks, fills B, .., n - B*(nb-1);
  * reserve(blocks, L, n): new list shares the old blocks (incref); if L % B
    != 0 the tail is written in place when fill[tail] == L % B, otherwise it
    is copied into a fresh block (cow = (tail, new, L % B)); the claimed
    fill is min(B, L % B + n); further blocks are fresh;
  * settle(blocks, L, n_res, n_act): free the reserved blocks past
    ceil((L+n_act)/B), lower the written tail's fill to what was written.
"""

from __future__ import annotations

import heapq


class PagedAllocRef:
    def __init__(self, num_blocks: int, block_size: int):
        self.nb = num_blocks
        self.bs = block_size
        self.ref = [0] * num_blocks
        self.fill = [0] * num_blocks
        self.heap = list(range(num_blocks))
        heapq.heapify(self.heap)

    def _blocks_for(self, n: int) -> int:
        return -(-n // self.bs)

    def _take(self) -> int:
        if not self.heap:
            raise MemoryError("KV pool out of blocks")
        b = heapq.heappop(self.heap)
        self.ref[b] = 1
        self.fill[b] = 0
        return b

    def _decref(self, b: int) -> None:
        assert self.ref[b] > 0, f"block {b} is not allocated"
        self.ref[b] -= 1
        if self.ref[b] == 0:
            self.fill[b] = 0
            heapq.heappush(self.heap, b)

    def alloc_seq(self, n: int) -> list[int]:
        nb = self._blocks_for(n)
        if len(self.heap) < nb:
            raise MemoryError("KV pool out of blocks")
        out = []
        for i in range(nb):
            b = self._take()
            self.fill[b] = min(self.bs, n - i * self.bs)
            out.append(b)
        return out

    def incref(self, blocks) -> None:
        for b in blocks:
            assert self.ref[b] > 0
        for b in blocks:
            self.ref[b] += 1

    def decref(self, blocks) -> None:
        for b in blocks:
            self._decref(b)

    def reserve(self, blocks, seq_len: int, n_new: int):
        bs = self.bs
        nb_old = self._blocks_for(seq_len)
        nb_new = self._blocks_for(seq_len + n_new)
        off = seq_len % bs
        tail = blocks[nb_old - 1]
        cow_needed = off != 0 and n_new > 0 and self.fill[tail] != off
        need = (nb_new - nb_old) + int(cow_needed)
        if len(self.heap) < need:
            raise MemoryError("KV pool out of blocks")
        out = list(blocks[:nb_old])
        for b in out:
            self.ref[b] += 1
        cow = [-1, -1, 0]
        if off != 0 and n_new > 0:
            dst = tail
            if cow_needed:
                dst = self._take()
                self._decref(tail)
                out[nb_old - 1] = dst
                cow = [tail, dst, off]
            self.fill[dst] = min(bs, off + n_new)
        remaining = seq_len + n_new - nb_old * bs
        for _ in range(nb_old, nb_new):
            b = self._take()
            self.fill[b] = min(bs, remaining)
            remaining -= bs
            out.append(b)
        return out, cow

    def settle(self, blocks, seq_len: int, n_res: int, n_act: int) -> list[int]:
        nb_res = self._blocks_for(seq_len + n_res)
        nb_act = self._blocks_for(seq_len + n_act)
        for b in blocks[nb_act:nb_res]:
            self._decref(b)
        if n_act < n_res:
            nb_old = self._blocks_for(seq_len)
            if nb_act > nb_old or seq_len % self.bs != 0:
                self.fill[blocks[nb_act - 1]] = seq_len + n_act - (nb_act - 1) * self.bs
        return list(blocks[:nb_act])

    def snapshot(self):
        return list(self.ref), list(self.fill), sorted(self.heap)

    def slot_mapping(self, blocks, start: int, count: int) -> list[int]:
        return [blocks[p // self.bs] * self.bs + p % self.bs for p in range(start, start + count)]
