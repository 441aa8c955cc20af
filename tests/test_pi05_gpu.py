"""F2 (pi0.5-shaped, bf16 on tcgen05) vs the torch-fp32 CPU oracle
(oracle/pi05_ref.py) at a reduced shape that runs the same kernels, plus the
reference's route-equality suites on the F2 backend and a full-shape run.

Tolerances (bf16 mode): KV and actions within 3e-2 of the
oracle's max magnitude; logits cosine >= 0.999; greedy tokens compared where
the oracle's top-2 margin exceeds the logit error bound (else reported)."""

import numpy as np
import pytest

from paper_2603_14371_b200 import BatchedState, BackendConfig, Observation
from paper_2603_14371_b200.verify import (suite_batching, suite_reference, suite_resumption,
                                          suite_sharing)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    from oracle.pi05_ref import Pi05Ref
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    be = Pi05Backend(TINY, num_blocks=256)
    return be, Pi05Ref.from_backend(be)


def _obs(n_img, toks, seed=11):
    from paper_2603_14371_b200.pi05 import Pi05Observation, synthetic_images
    return Pi05Observation(tuple(toks), 0, synthetic_images(n_img, seed) if n_img else None)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-9))


def test_weight_init_is_the_splitmix_counter(tiny):
    be, ref = tiny
    ref.check_init(be, names=("embed", "llm.0.wqkv", "mod.b", "vit.0.ln1.w", "action_out"))


@pytest.mark.parametrize("n_img, toks", [(0, (5, 17, 99, 3)), (1, (7, 8)), (2, tuple(range(40, 110)))])
def test_prefill_kv_matches_oracle(tiny, n_img, toks):
    be, ref = tiny
    obs = _obs(n_img, toks)
    kv = be.prefill(obs)
    assert kv.seq_len == 256 * n_img + len(toks)
    want = ref.prefill(obs)
    for l, layer in enumerate(kv.layers):
        assert rel(layer.keys, want[l][0].numpy()) < 3e-2, l
        assert rel(layer.values, want[l][1].numpy()) < 3e-2, l


def test_action_denoise_matches_oracle(tiny):
    be, ref = tiny
    obs = _obs(1, (3, 4, 5))
    kv = be.prefill(obs)
    got = be.action_denoise(kv, be.config.S).actions
    want = ref.denoise(ref.prefill(obs), be.config.S)
    assert got.shape == (be.config.H, be.config.action_dim)
    assert rel(got, want) < 3e-2


def test_decode_logits_and_tokens_match_oracle(tiny):
    be, ref = tiny
    obs = _obs(1, (9, 10, 11, 12))
    kv = be.prefill(obs)
    out, logits = be.batched_language_decode(
        BatchedState((kv,), ((),), (False,), (0,), (6,), (0,)), 6, return_logits=True)
    import torch
    dev_kv = [tuple(torch.tensor(x, dtype=torch.float32) for x in be.read_kv(kv, l))
              for l in range(be.config.depth)]
    toks, _, want_logits = ref.decode(dev_kv, (), 6)  # the device prefix: decode numerics alone
    got = out.token_buffers[0]
    n = min(len(got), len(toks))
    for s in range(n):
        if got[:s] != toks[:s]:
            break  # diverged on an earlier near-tie: later steps see different inputs
        a, b = logits[s, 0].astype(np.float64), want_logits[s].astype(np.float64)
        cos = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
        assert cos > 0.9999, (s, cos)
        top2 = np.sort(b)[-2:]
        if top2[1] - top2[0] > 2 * np.max(np.abs(a - b)):
            assert got[s] == toks[s], (s, got, toks)


def test_kv_pool_shared_between_action_and_language(tiny):
    be, _ = tiny
    kv = be.prefill(_obs(1, (1, 2, 3)))
    snap = [(l.keys.copy(), l.values.copy()) for l in kv.layers]
    a1 = be.action_denoise(kv, be.config.S)
    for (k0, v0), layer in zip(snap, kv.layers):
        assert np.array_equal(k0, layer.keys) and np.array_equal(v0, layer.values)
    a2 = be.action_denoise(kv, be.config.S)
    assert a1 == a2


def test_batched_admission_matches_single(tiny):
    be, _ = tiny
    from paper_2603_14371_b200.workload import Arrival
    arr = [Arrival(0, _obs(1, (4, 5, i + 6), seed=20 + i), 3) for i in range(3)]
    got = be.admit_many(arr, 0)
    for (chunk, st), a in zip(got, arr):
        solo = be.action_denoise(be.prefill(a.observation), be.config.S)
        assert rel(chunk.actions, solo.actions) < 2e-2
        assert st.kv.seq_len == 256 + 3


def test_batch_invariant_decode(tiny):
    be, _ = tiny
    caches = [be.prefill(_obs(0, (i + 2, i + 3, 7))) for i in range(4)]
    big = be.batched_language_decode(
        BatchedState(tuple(caches), ((),) * 4, (False,) * 4, (0, 1, 2, 3), (5,) * 4, (0,) * 4), 5)
    for i, kv in enumerate(caches):
        solo = be.batched_language_decode(
            BatchedState((kv,), ((),), (False,), (i,), (5,), (0,)), 5)
        assert big.token_buffers[i] == solo.token_buffers[0]
        assert big.kv_batch[i] == solo.kv_batch[0]


def test_cuda_graph_replay_is_bit_identical(tiny):
    """Calls 1 (eager), 2 (captured) and 3+ (replayed) of one shape agree exactly."""
    be, _ = tiny
    obs = _obs(1, (21, 22, 23))
    kvs = [be.prefill(obs) for _ in range(4)]
    for kv in kvs[1:]:
        assert kv == kvs[0]
    acts = [be.action_denoise(kvs[0], be.config.S) for _ in range(4)]
    assert all(a == acts[0] for a in acts)
    outs = [be.batched_language_decode(
        BatchedState((kv,), ((),), (False,), (0,), (7,), (0,)), 7) for kv in kvs]
    for out in outs[1:]:
        assert out.token_buffers == outs[0].token_buffers
        assert out.kv_batch[0] == outs[0].kv_batch[0]


@pytest.mark.parametrize("rows, ctxs", [(1, [1]), (3, [64, 65, 130]), (5, [800, 805, 37, 1024, 2000]),
                                        (64, [1024] * 64)])
def test_paged_decode_attention_matches_torch(rows, ctxs):
    """Kernel-level parity on identical paged data: 8 query heads over 1 KV head,
    keys [0, pos] gathered through a random block table (torch fp32 reference)."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(rows)
    maxb = max((c + 63) // 64 for c in ctxs)
    nb = rows * maxb + 3
    kp = (torch.randn(nb, 64, 256, generator=g) * 0.5).to(torch.bfloat16).cuda()
    vp = torch.randn(nb, 64, 256, generator=g).to(torch.bfloat16).cuda()
    bt = torch.randperm(nb, generator=g)[: rows * maxb].reshape(rows, maxb).to(torch.int32).cuda()
    pos = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32).cuda()
    q = torch.randn(rows, 2048, generator=g).to(torch.bfloat16).cuda()
    out = torch.empty_like(q)
    ws = torch.empty(rows * maxb * 8 * 258, dtype=torch.float32, device="cuda")
    for _ in range(2):  # second call reuses the self-resetting merge counters
        _lib.call("oxy_paged_decode_attention", C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
                  C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()),
                  C.c_int32(maxb), C.c_void_p(pos.data_ptr()), C.c_int32(rows), C.c_int32(maxb),
                  C.c_void_p(ws.data_ptr()), _lib.stream_ptr())
        torch.cuda.synchronize()
    for r, c in enumerate(ctxs):
        idx = bt[r].long()
        K = kp[idx].reshape(-1, 256)[:c].float()
        V = vp[idx].reshape(-1, 256)[:c].float()
        qh = q[r].float().reshape(8, 256)
        ref = torch.softmax(qh @ K.T / 16.0, -1) @ V
        torch.testing.assert_close(out[r].float().reshape(8, 256), ref, atol=2e-2, rtol=2e-2)


def _pi05_factory(cfg: BackendConfig):
    from paper_2603_14371_b200.pi05 import Pi05Backend
    return Pi05Backend(cfg, num_blocks=128)


@pytest.mark.parametrize("suite, n", [(suite_batching, 6), (suite_resumption, 8), (suite_sharing, 5),
                                      (suite_reference, 10)])
def test_reference_suites_on_pi05_backend(suite, n):
    rep = suite(n, backend_factory=_pi05_factory)
    assert rep.ok, rep.failures[:3]


def test_full_shape_frame_runs():
    """The BASELINE config-2 shape: 3 cameras + 32 prompt tokens, chunk 50."""
    from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config
    be = Pi05Backend(Pi05Config(), num_blocks=256)
    obs = _obs(3, tuple(range(1000, 1032)))
    kv = be.prefill(obs)
    assert kv.seq_len == 800
    chunk = be.action_denoise(kv, 10)
    assert chunk.actions.shape == (50, 32) and np.all(np.isfinite(chunk.actions))
    out = be.batched_language_decode(BatchedState((kv,), ((),), (False,), (0,), (5,), (0,)), 5)
    assert len(out.token_buffers[0]) == 5 and out.kv_batch[0].seq_len == 805
    k0 = out.kv_batch[0].layers[0].keys
    assert np.all(np.isfinite(k0)) and np.abs(k0).max() > 0


@pytest.mark.parametrize("pattern", ["OnePerFrame", "Poisson"])
def test_overlapped_frames_match_stage_serial(pattern):
    """Denoise on the action-expert lane overlapping the batched decode gives
    the same transcript (actions, tokens, completion frames) as running the
    stages back to back, and the measured frame time is no more than the sum."""
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    from paper_2603_14371_b200.sim_engine import SimConfig, run_simulation, transcript_to_json
    from paper_2603_14371_b200.workload import WorkloadSpec
    cfg = SimConfig(backend_kind="Pi05", backend_config=BackendConfig(vocab=TINY.vocab),
                    workload=WorkloadSpec(pattern=pattern, default_N=9, obs_len=24, num_frames=8,
                                          seed=5, lam=1.5),
                    k=3)
    runs = {}
    for overlap in (False, True):
        be = Pi05Backend(TINY, num_blocks=256, measure=True, overlap=overlap)
        runs[overlap] = run_simulation(cfg, backend=be)
    assert transcript_to_json(runs[True]) == transcript_to_json(runs[False])
    for tr in runs[True].traces:
        if tr.arrival_count:
            assert 0 < tr.total_us <= sum(tr.latency_components) + 2000, tr


def test_extra_tasks_share_prefix_blocks_with_copy_on_write():
    """Two language tasks on one observation (Arrival.extra_tasks): one prefill,
    the prefix blocks refcounted by both requests, the shared tail block copied
    on the first decoded token, and each task's tokens equal to a solo decode
    of the same prefix (batch-invariant kernels)."""
    from paper_2603_14371_b200 import Arrival, KvManager
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    from paper_2603_14371_b200.scheduler import run_frame_unified
    be = Pi05Backend(TINY, num_blocks=64)
    obs = _obs(1, tuple(range(20, 50)))  # 286 positions: 4 full blocks + a partially filled tail
    free0 = be.allocator.num_free
    mgr = KvManager()
    res = run_frame_unified(0, [Arrival(0, obs, 6, extra_tasks=(6,))], mgr, be, 3, 30.0)
    assert res.trace.prefill_count == 1 and res.trace.batch_size_m == 2
    a, b = (mgr.retrieve(r) for r in mgr.active_ids())
    assert a.tokens == b.tokens and len(a.tokens) == 3
    assert a.kv.blocks[-1] != b.kv.blocks[-1]  # the tail block was copied on write ...
    assert a.kv.blocks[:-1] == b.kv.blocks[:-1]  # ... the full prefix blocks are shared
    nb = be.allocator.blocks_for(286 + 3)
    assert free0 - be.allocator.num_free == nb + 1  # one prefix + one copied tail, not two prefixes
    solo_kv = be.prefill(obs)
    solo = be.batched_language_decode(BatchedState((solo_kv,), ((),), (False,), (0,), (6,), (0,)), 3)
    assert solo.token_buffers[0] == a.tokens
    del solo, solo_kv, a, b
    for r in list(mgr.active_ids()):
        mgr.remove(r)
    import gc
    gc.collect()
    assert be.allocator.num_free == free0


def test_cross_variant_invariance_on_pi05_backend():
    """The reference's acceptance criterion 3 (tests/test_acceptance.py:81-113) on
    the pi0.5 backend: Unified, SharedNoBatch and IsolatedSequential produce the
    same request set, greedy tokens and action chunks (exact equality), because
    every kernel is batch-invariant and deterministic."""
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    from paper_2603_14371_b200.rng import SplitMix64
    from paper_2603_14371_b200.sim_engine import SimConfig, run_simulation
    from paper_2603_14371_b200.workload import WorkloadSpec
    rng = SplitMix64(2026)
    be = Pi05Backend(TINY, num_blocks=512)
    compared = 0
    for i in range(4):
        pattern = ("OnePerFrame", "Uniform", "Poisson", "MixedLength")[i]
        wl = WorkloadSpec(pattern=pattern, default_N=2 + rng.below(9), obs_len=2 + rng.below(9),
                          num_frames=4 + rng.below(5), seed=rng.below(1 << 32), lam=0.25 + rng.uniform(),
                          r=1 + rng.below(2), short_N=2 + rng.below(5), long_N=8 + rng.below(6),
                          p_long=rng.uniform())
        k = 1 + rng.below(6)
        bc = BackendConfig(vocab=TINY.vocab)
        runs = {v: run_simulation(SimConfig(variant=v, backend_kind="Pi05", backend_config=bc, workload=wl, k=k),
                                  backend=be)
                for v in ("Unified", "SharedNoBatch", "IsolatedSequential")}
        base = runs["Unified"].transcript
        for v in ("SharedNoBatch", "IsolatedSequential"):
            other = runs[v].transcript
            assert sorted(other) == sorted(base), (i, v)
            for rid, entry in base.items():
                assert other[rid].tokens == entry.tokens, (i, v, rid)
                assert other[rid].action == entry.action, (i, v, rid)
                compared += 1
    assert compared > 0


def test_decode_budget_below_k_across_block_boundary(tiny):
    """seq + k crosses a 64-slot block, seq + remaining budget does not: the row
    reserves min(k, budget) positions and the call must accept the shorter table."""
    be, _ = tiny
    kv = be.prefill(_obs(0, tuple(range(2, 62))))  # P = 60: one block
    out = be.batched_language_decode(BatchedState((kv,), ((),), (False,), (0,), (2,), (0,)), 8)
    n = len(out.token_buffers[0])
    assert 1 <= n <= 2 and out.kv_batch[0].seq_len == 60 + n
    assert len(out.kv_batch[0].blocks) == 1


def test_abi_rejects_block_ids_outside_the_pool(tiny):
    """A non-Python host cannot make the pi0.5 entry points touch memory past the
    pool: every block id is checked against the pool size (OXY_EINVAL)."""
    import ctypes as C
    from paper_2603_14371_b200 import _lib
    be, _ = tiny
    nb = be.allocator.num_blocks
    toks = _lib.as_i32([5, 6, 7])
    for bad in (nb, -1, 1 << 20):
        blocks = _lib.as_i32([bad])
        with pytest.raises(ValueError, match="outside pool"):
            _lib.call("oxy_pi05_prefill", be._h, C.c_int32(1), _lib.ptr_i32(_lib.as_i32([0])),
                      _lib.ptr_i32(_lib.as_i32([3])), _lib.ptr_i32(toks), None, _lib.ptr_i32(blocks),
                      _lib.stream_ptr())
        with pytest.raises(ValueError, match="outside pool"):
            _lib.call("oxy_pi05_denoise_async", be._h, C.c_int32(1), _lib.ptr_i32(_lib.as_i32([3])),
                      _lib.ptr_i32(blocks), C.c_int32(2), None, _lib.stream_ptr())
        out = np.zeros(4, np.int32)
        with pytest.raises(ValueError, match="outside pool"):
            _lib.call("oxy_pi05_decode", be._h, C.c_int32(1), C.c_int32(1), _lib.ptr_i32(blocks),
                      C.c_int32(1), _lib.ptr_i32(_lib.as_i32([3])), _lib.ptr_i32(_lib.as_i32([1])),
                      _lib.ptr_i32(_lib.as_i32([1])), _lib.ptr_i32(_lib.as_i32([-1, -1, 0])),
                      _lib.ptr_i32(out), _lib.ptr_i32(out), None, _lib.stream_ptr())
        with pytest.raises(ValueError, match="outside pool"):
            _lib.call("oxy_pi05_decode", be._h, C.c_int32(1), C.c_int32(1), _lib.ptr_i32(_lib.as_i32([0])),
                      C.c_int32(1), _lib.ptr_i32(_lib.as_i32([3])), _lib.ptr_i32(_lib.as_i32([1])),
                      _lib.ptr_i32(_lib.as_i32([1])), _lib.ptr_i32(_lib.as_i32([0, bad, 3])),
                      _lib.ptr_i32(out), _lib.ptr_i32(out), None, _lib.stream_ptr())
        keys = np.zeros((3, 256), np.float32)
        with pytest.raises(ValueError, match="outside pool"):
            _lib.call("oxy_pi05_read_kv", be._h, _lib.ptr_i32(blocks), C.c_int32(3), C.c_int32(0),
                      keys.ctypes.data_as(C.c_void_p), keys.ctypes.data_as(C.c_void_p), _lib.stream_ptr())


def test_failed_decode_reservation_leaves_the_pool_unchanged():
    """Pool exhaustion part-way through a batch's reservations rolls back the rows
    already reserved (blocks, copy-on-write copies, tail watermarks): the allocator
    state after the MemoryError equals the state before the call."""
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    be = Pi05Backend(TINY, num_blocks=6)
    a = be.prefill(_obs(0, tuple(range(2, 40))))    # 1 block, tail partially filled
    b = be.prefill(_obs(0, tuple(range(2, 130))))   # 3 blocks
    snap = be.allocator.snapshot()
    # row 0 shares a's tail with row 1 (copy-on-write), row 2 needs more blocks than are left
    with pytest.raises(MemoryError):
        be.batched_language_decode(BatchedState((a, a, b), ((),) * 3, (False,) * 3, (0, 1, 2),
                                                (200,) * 3, (0,) * 3), 150)
    after = be.allocator.snapshot()
    for x, y in zip(snap, after):
        assert np.array_equal(x, y)


def test_recompute_logits_matches_cached_decode(tiny):
    """The no-cache route (dense forward, prefix-LM mask, plain fp32 attention) and
    the cached paged decode agree on every step's logits of a 4-step decode."""
    be, _ = tiny
    obs = _obs(1, (31, 32, 33))
    kv = be.prefill(obs)
    out, logits = be.batched_language_decode(
        BatchedState((kv,), ((),), (False,), (0,), (4,), (0,)), 4, return_logits=True)
    toks = out.token_buffers[0]
    # image positions are not token ids: recompute covers token-only prefixes, so use
    # a token-only observation for the route comparison
    kv2 = be.prefill(_obs(0, (31, 32, 33, 34, 35)))
    out2, logits2 = be.batched_language_decode(
        BatchedState((kv2,), ((),), (False,), (0,), (4,), (0,)), 4, return_logits=True)
    seq = [31, 32, 33, 34, 35, be.config.eos_token]
    for s, t in enumerate(out2.token_buffers[0]):
        want = be.recompute_logits(seq)
        got = logits2[s, 0].astype(np.float64)
        cos = got @ want / (np.linalg.norm(got) * np.linalg.norm(want))
        assert cos > 0.9999, (s, cos)
        assert int(np.argmax(want)) == t or np.sort(want)[-1] - np.sort(want)[-2] < 2 * np.abs(got - want).max()
        seq.append(t)
    assert len(toks) >= 1


def test_pool_exhaustion_fails_at_admission_not_in_decode():
    """With a pool too small for every arrival's full decode, the frame that cannot
    be covered fails while admitting (its prefix or its decode budget does not fit
    in the blocks not promised to live requests); the decodes of requests already
    admitted never run out of blocks."""
    from paper_2603_14371_b200 import Arrival, KvManager
    from paper_2603_14371_b200.pi05 import TINY, Pi05Backend
    from paper_2603_14371_b200.scheduler import run_frame_unified
    be = Pi05Backend(TINY, num_blocks=12)
    mgr = KvManager()
    admitted_frames = 0
    with pytest.raises(MemoryError, match="not promised"):
        for t in range(40):
            run_frame_unified(t, [Arrival(t, _obs(0, tuple(range(3, 63)), seed=t), 200)], mgr, be, 8, 30.0)
            admitted_frames += 1
    assert admitted_frames >= 2
    # the live requests keep decoding to their budgets without touching the limit
    for t in range(40, 80):
        if not mgr.active_ids():
            break
        run_frame_unified(t, [], mgr, be, 8, 30.0)
    assert be.allocator.promised >= 0
