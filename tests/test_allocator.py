"""The C++ paged-KV allocator (through the C ABI) is bit-exact with its
Python restatement (oracle/paged_alloc.py) under random op walks that mimic
the scheduler: prefill, decode reserve/settle (including forks of one state
decoded twice, which force copy-on-write), handle drops."""

import os

import numpy as np
import pytest

from conftest import ROOT
from oracle.paged_alloc import PagedAllocRef
from paper_2603_14371_b200 import _lib
from paper_2603_14371_b200.rng import SplitMix64

pytestmark = pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="extension not built")


def _alloc(nb, bs):
    from paper_2603_14371_b200.paged import BlockAllocator
    return BlockAllocator(nb, bs)


def _same_state(a, r):
    ref, fill, free = a.snapshot()
    rr, rf, rfree = r.snapshot()
    assert ref.tolist() == rr
    assert fill.tolist() == rf
    assert free.tolist() == rfree


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/oxygen_b200.h but not exported"


def test_prefill_and_lowest_id_first():
    a, r = _alloc(16, 4), PagedAllocRef(16, 4)
    assert a.alloc_seq(9) == tuple(r.alloc_seq(9)) == (0, 1, 2)
    assert a.alloc_seq(4) == tuple(r.alloc_seq(4)) == (3,)
    a.decref((1,))
    r.decref([1])
    assert a.alloc_seq(1) == tuple(r.alloc_seq(1)) == (1,)
    _same_state(a, r)


def test_in_place_then_cow_on_fork():
    a, r = _alloc(16, 4), PagedAllocRef(16, 4)
    base = a.alloc_seq(6)
    r.alloc_seq(6)
    # first extension of the shared state writes the tail in place
    b1, cow1 = a.reserve(base, 6, 3)
    rb1, rcow1 = r.reserve(list(base), 6, 3)
    assert b1.tolist() == rb1 and cow1.tolist() == rcow1 == [-1, -1, 0]
    # second extension of the same state must copy the tail (slots 0..1)
    b2, cow2 = a.reserve(base, 6, 2)
    rb2, rcow2 = r.reserve(list(base), 6, 2)
    assert b2.tolist() == rb2 and cow2.tolist() == rcow2
    assert cow2[0] == base[1] and cow2[2] == 2
    _same_state(a, r)


def test_slot_mapping():
    a, r = _alloc(8, 4), PagedAllocRef(8, 4)
    blocks = (5, 2, 7)
    assert a.slot_mapping(blocks, 0, 12).tolist() == r.slot_mapping(blocks, 0, 12)
    assert a.slot_mapping(blocks, 0, 5).tolist() == [20, 21, 22, 23, 8]


def test_out_of_blocks_raises_without_corrupting():
    a, r = _alloc(3, 4), PagedAllocRef(3, 4)
    a.alloc_seq(8)
    r.alloc_seq(8)
    with pytest.raises(MemoryError, match="out of blocks"):
        a.alloc_seq(5)
    _same_state(a, r)


def test_bad_block_id_rejected():
    a = _alloc(4, 4)
    with pytest.raises(ValueError, match="outside pool"):
        a.decref((9,))
    with pytest.raises(RuntimeError, match="not allocated"):
        a.decref((0,))


@pytest.mark.parametrize("seed", range(12))
def test_random_walks_bit_exact(seed):
    rng = SplitMix64(9000 + seed)
    bs = (1, 2, 4, 16)[seed % 4]
    nb = 400
    a, r = _alloc(nb, bs), PagedAllocRef(nb, bs)
    handles = []  # (blocks, seq_len), owned by the walk
    for step in range(250):
        op = rng.below(100)
        if op < 25 or not handles:
            n = 1 + rng.below(3 * bs + 2)
            got = a.alloc_seq(n)
            assert list(got) == r.alloc_seq(n)
            handles.append((list(got), n))
        elif op < 70:
            # decode: reserve n_res, run, settle n_act (the fork keeps the parent)
            i = rng.below(len(handles))
            blocks, L = handles[i]
            n_res = 1 + rng.below(2 * bs + 1)
            n_act = 1 + rng.below(n_res)
            nb_, cow = a.reserve(blocks, L, n_res)
            rnb, rcow = r.reserve(blocks, L, n_res)
            assert nb_.tolist() == rnb, f"step {step}"
            assert cow.tolist() == rcow, f"step {step}"
            kept = a.settle(nb_, L, n_res, n_act)
            assert list(kept) == r.settle(rnb, L, n_res, n_act)
            handles.append((list(kept), L + n_act))
            if rng.below(2):  # scheduler path: the old state is replaced
                old = handles.pop(i)
                a.decref(old[0])
                r.decref(old[0])
        else:
            i = rng.below(len(handles))
            blocks, _ = handles.pop(i)
            a.decref(blocks)
            r.decref(blocks)
        _same_state(a, r)
    for blocks, _ in handles:
        a.decref(blocks)
        r.decref(blocks)
    _same_state(a, r)
    assert a.num_free == nb


class _Owner:
    """Minimal backend stand-in for PagedKvCache on the CPU (allocator only)."""
    backend_tag = "alloc-test"
    num_layers = 1

    def __init__(self, num_blocks, block_size):
        from paper_2603_14371_b200.paged import BlockAllocator
        self.allocator = BlockAllocator(num_blocks, block_size)


def _decode(owner, handles, n_new, n_written):
    """What a backend's batched decode does around its kernel: reserve -> settle -> carry."""
    from paper_2603_14371_b200.paged import PagedKvCache
    a = owner.allocator
    tables, cows, drawn = a.reserve_rows(handles, n_new)
    news = [PagedKvCache(owner, a.settle(t, h.seq_len, n, w), h.seq_len + w)
            for t, h, n, w in zip(tables, handles, n_new, n_written)]
    a.carry_promises(handles, news, drawn)
    return news


def test_admission_budget_keeps_decode_from_running_out():
    """The reference checks capacity only at store (kvweaver/kv_manager.py:195-238)
    and decode growth never fails.  Admission sets aside every block a request's
    decode can take; allocations without a promise only use unpromised blocks and
    fail up front, leaving the allocator untouched."""
    from paper_2603_14371_b200.paged import PagedKvCache
    owner = _Owner(10, 4)
    a = owner.allocator
    h = PagedKvCache(owner, a.alloc_seq(6), 6)            # 2 blocks, tail holds 2 of 4 slots
    a.promise_budget(h, 10)                                # ceil(16/4) - 2 + 1 copy-on-write = 3
    assert a.promised == 3 and a.unpromised_free() == 5
    with pytest.raises(MemoryError, match="not promised"):
        a.alloc_seq(24)                                    # 6 blocks > 5 unpromised
    [h2] = _decode(owner, [h], [4], [4])                   # 1 new block, drawn from the promise
    assert h2.seq_len == 10 and len(h2.blocks) == 3 and h2.promise == 2 and a.promised == 2
    filler = PagedKvCache(owner, a.alloc_seq(20), 20)     # every unpromised block taken
    assert a.unpromised_free() == 0 and a.num_free == 2
    snap = a.snapshot()
    with pytest.raises(MemoryError, match="decode row"):
        _decode(owner, [h], [4], [4])                      # a fork of the old state: no promise left
    for x, y in zip(snap, a.snapshot()):
        assert np.array_equal(x, y)
    [h3] = _decode(owner, [h2], [6], [6])                  # the admitted request still grows
    assert h3.seq_len == 16 and a.num_free == 1 and a.promised == h3.promise == 1
    del h, h2, h3, filler
    import gc
    gc.collect()
    assert a.promised == 0 and a.num_free == 10
