"""Host layers (manager, scheduler, driver, metrics, suites) on the CPU with the
cost backend: identical traces and summaries to the reference
(tests/golden/sim.json), the reference's error messages, and the
model-free oracle suites."""

import numpy as np
import pytest

from paper_2603_14371_b200 import (BatchedState, CostModelParams, GenerationState, KvCache,
                                   KvLayer, KvManager, Observation, SimConfig, WorkloadSpec,
                                   make_backend, run_simulation, speedup, summarize)
from paper_2603_14371_b200.backend import ActionChunk, BackendConfig
from paper_2603_14371_b200.scheduler import (FrameTrace, run_frame_isolated_parallel,
                                             run_frame_isolated_sequential,
                                             run_frame_shared_no_batch, run_frame_unified)
from paper_2603_14371_b200.sim_engine import SimResult
from paper_2603_14371_b200.verify import suite_cost, suite_littles_law, suite_manager
from paper_2603_14371_b200.workload import Arrival

TAG = "toy/test"


def cache(n, layers=2, fill=0.5):
    return KvCache(tuple(KvLayer(np.full((n, 8), fill + i), np.full((n, 8), fill - i))
                         for i in range(layers)), n, TAG)


def state(n=4, tokens=(), max_len=10, terminated=False):
    return GenerationState(cache(n), tokens, terminated, 0, max_len)


class TestValueObjects:
    def test_read_only_and_shape(self):
        l = KvLayer(np.zeros((3, 8)), np.zeros((3, 8)))
        with pytest.raises(ValueError):
            l.keys[0, 0] = 1.0
        with pytest.raises(ValueError, match="matching 2-d"):
            KvLayer(np.zeros((3, 8)), np.zeros((4, 8)))

    def test_cache_checks(self):
        good = KvLayer(np.zeros((3, 8)), np.zeros((3, 8)))
        bad = KvLayer(np.zeros((2, 8)), np.zeros((2, 8)))
        with pytest.raises(ValueError, match="layer 1 reports seq_len 2"):
            KvCache((good, bad), 3, TAG)
        with pytest.raises(ValueError, match="at least one layer"):
            KvCache((), 0, TAG)
        assert cache(3) == cache(3) and cache(3) != cache(3, fill=0.7)

    def test_generation_state_invariants(self):
        with pytest.raises(ValueError, match="must be terminated"):
            state(6, (1, 2), max_len=2)
        with pytest.raises(ValueError, match="must have emitted"):
            state(4, (), terminated=True)
        with pytest.raises(ValueError, match="cannot hold"):
            state(1, (1, 2), max_len=5)
        assert state(6, (1, 2)).prefill_len == 4

    def test_action_chunk(self):
        with pytest.raises(ValueError, match="non-finite"):
            ActionChunk(np.array([[np.inf, 0.0]]))
        a = ActionChunk(np.ones((2, 3)))
        assert a == ActionChunk(np.ones((2, 3))) and a.horizon == 2

    def test_backend_config_validation(self):
        with pytest.raises(ValueError, match="not divisible"):
            BackendConfig(d_model=30, n_heads=4)
        with pytest.raises(ValueError, match="outside vocab"):
            BackendConfig(vocab=4, eos_token=4)


class TestManager:
    def test_lifecycle_and_messages(self):
        m = KvManager()
        assert [m.store(state()) for _ in range(3)] == [0, 1, 2]
        m.remove(1)
        assert m.store(state()) == 3 and m.active_ids() == [0, 2, 3]
        with pytest.raises(KeyError, match="unknown request id 9"):
            m.retrieve(9)
        with pytest.raises(KeyError, match="unknown request id 1"):
            m.remove(1)
        with pytest.raises(ValueError, match="terminated"):
            m.store(state(5, (1,), terminated=True))

    def test_update_checks(self):
        m = KvManager()
        rid = m.store(state(4, (1,)))
        m.update(rid, GenerationState(cache(5), (1, 2), False, 0, 10))
        with pytest.raises(ValueError, match="drops decoded tokens"):
            m.update(rid, GenerationState(cache(6), (9, 2, 3), False, 0, 10))
        with pytest.raises(ValueError, match="shrinks the cache"):
            m.update(rid, GenerationState(cache(4), (1, 2), False, 0, 10))
        with pytest.raises(ValueError, match="prefill length changed"):
            m.update(rid, GenerationState(cache(7), (1, 2, 3), False, 0, 10))
        other = GenerationState(KvCache((6, 6), 6, "other"), (1, 2, 3), False, 0, 10)
        with pytest.raises(ValueError, match="switches backend"):
            m.update(rid, other)

    def test_capacity_and_gauge(self):
        m = KvManager(capacity_positions=10)
        m.store(state(4))
        m.store(state(6))
        assert m.live_positions == 10
        with pytest.raises(ValueError, match="capacity exceeded"):
            m.store(state(1))

    def test_batching(self):
        m = KvManager()
        with pytest.raises(ValueError, match="zero requests"):
            m.batch([], [])
        with pytest.raises(ValueError, match="request 7 is terminated"):
            m.batch([state(5, (1,), terminated=True)], [7])
        with pytest.raises(ValueError, match="2 states but 1 ids"):
            m.batch([state(), state()], [0])
        with pytest.raises(ValueError, match="flags has 2"):
            BatchedState((cache(2),), ((),), (False, False), (0,), (3,), (0,))
        sts = [state(3 + i, tuple(range(i))) for i in range(4)]
        assert m.unbatch(m.batch(sts, [4, 5, 6, 7])) == sts

    def test_manager_suite(self):
        rep = suite_manager(1000, seed=41105)
        assert rep.ok, rep.failures[:2]


def _trace_rows(res):
    return [[t.frame, list(t.latency_components), t.batch_size_m, t.tokens_emitted,
             t.actions_emitted, list(t.completed_ids), t.deadline_met, t.total_us,
             t.arrival_count] for t in res.traces]


class TestCostModelSimulation:
    def test_traces_and_summaries_match_reference(self, golden):
        for case in golden("sim.json")["cost"]:
            cfg = SimConfig(variant=case["variant"], backend_kind="CostModel",
                            cost_params=CostModelParams(),
                            workload=WorkloadSpec(**case["workload"]), k=case["k"])
            res = run_simulation(cfg)
            assert _trace_rows(res) == case["traces"], case["variant"]
            rep = summarize(res, cfg)
            assert [getattr(rep, f) for f in rep.__slots__] == case["summary"]
            rep = summarize(res, cfg, include_warmup=True)
            assert [getattr(rep, f) for f in rep.__slots__] == case["summary_full"]

    def test_steady_state_closed_form(self):
        cost = CostModelParams()
        wl = dict(default_N=12, obs_len=800, num_frames=40)

        def rep(variant):
            cfg = SimConfig(variant=variant, backend_kind="CostModel", cost_params=cost,
                            workload=WorkloadSpec(**wl), k=4)
            res = run_simulation(cfg)
            return res, summarize(res, cfg)

        uni, ru = rep("Unified")
        for tr in uni.traces[2:40]:
            assert (tr.batch_size_m, tr.tokens_emitted, len(tr.completed_ids)) == (3, 12, 1)
        _, ri = rep("IsolatedSequential")
        assert abs(speedup(ru, ri) - 142_000 / 74_800) < 1e-9

    def test_cost_and_littles_law_suites(self):
        assert suite_cost().ok
        assert suite_littles_law(lams=(0.5,), frames=4000, tol=0.08).ok

    def test_scheduler_edge_cases(self):
        be = make_backend("CostModel", BackendConfig(), CostModelParams())
        m = KvManager()
        assert run_frame_unified(0, [], m, be, 4, 30.0).trace.total_us == 0
        with pytest.raises(ValueError, match="latency model"):
            class Fake:
                kind = "Toy"
            run_frame_isolated_parallel(0, [], Fake(), 30.0, 0)
        arr = [Arrival(0, Observation((1,) * 800, 0), 12)]
        res = run_frame_isolated_sequential(0, arr, be, 30.0, 5)
        assert res.trace.prefill_count == 2 and res.finished[0][0] == 5
        res = run_frame_shared_no_batch(0, arr, m, be, 30.0)
        assert res.trace.total_us == 20000 + 30000 + 12 * 6000

    @pytest.mark.parametrize("kw, msg", [
        (dict(variant="X"), "unknown variant"),
        (dict(backend_kind="X"), "unknown backend"),
        (dict(k=0), "k must be >= 1"),
        (dict(pacing="FixedPeriod"), "period_us"),
        (dict(variant="IsolatedParallel", backend_kind="Toy"), "latency-model only"),
    ])
    def test_sim_config_validation(self, kw, msg):
        with pytest.raises(ValueError, match=msg):
            SimConfig(**kw)


def test_metrics_hand_values():
    def tr(frame, total, tokens=0, actions=10, m=1):
        return FrameTrace(frame, 1, (0, 0, 0, 0), m, tokens, actions, (), True, total, 1)

    cfg = SimConfig(backend_kind="CostModel",
                    workload=WorkloadSpec(default_N=4, obs_len=10, num_frames=4), k=4)
    res = SimResult((tr(0, 200_000, 4), tr(1, 200_000, 4)), {})
    rep = summarize(res, cfg, include_warmup=True)
    assert rep.action_freq_hz == pytest.approx(50.0)
    assert rep.token_throughput == pytest.approx(20.0)
    with pytest.raises(ValueError, match="degenerate"):
        summarize(SimResult((tr(0, 0),), {}), cfg, include_warmup=True)


def test_cost_calibration_recovers_constants_and_trends():
    """calibrate.fit_cost_params inverts the cost model exactly on model-generated
    samples, and with B200-like constants the reference's sweep trends hold
    (tests/test_acceptance.py:145-200 shapes)."""
    from paper_2603_14371_b200.backend import CostModelParams
    from paper_2603_14371_b200.calibrate import closed_form_speedup, fit_cost_params
    true = CostModelParams(11, 870, 1300, 12, 1.0)
    pre = [(p, true.c_prefill_per_token * p) for p in (32, 288, 544, 800)]
    den = [(s, s * true.c_denoise_per_step) for s in (1, 5, 10)]
    dec = [(5, m, 5 * (true.c_decode_base + true.c_decode_per_request * m)) for m in (1, 2, 4, 8, 16)]
    assert fit_cost_params(pre, den, dec) == true
    # closed form of tests/test_acceptance.py:129-133 with the reference's constants
    ref = CostModelParams()
    assert abs(closed_form_speedup(ref, 12, 4, 800, 10) - 142000 / 74800) < 1e-12
    # unified beats isolated more as N grows, less as k grows
    s_n = [closed_form_speedup(true, n, 5, 800, 10) for n in (5, 10, 20, 30, 40)]
    s_k = [closed_form_speedup(true, 30, k, 800, 10) for k in (1, 2, 5, 10, 15, 30)]
    assert all(b > a for a, b in zip(s_n, s_n[1:]))
    assert all(b <= a for a, b in zip(s_k, s_k[1:]))


def test_csv_v1_row_matches_reference_format():
    """report.csv_row reproduces the reference CLI's v1 row (kvweaver/cli.py:80-101)
    for a cost-model run, value for value, against tests/golden/sim.json's
    summaries where available and the row schema otherwise."""
    from paper_2603_14371_b200 import SimConfig, WorkloadSpec, run_simulation, summarize
    from paper_2603_14371_b200.report import CSV_COLUMNS, csv_row, write_csv
    cfg = SimConfig(variant="Unified", backend_kind="CostModel", k=4,
                    workload=WorkloadSpec(pattern="OnePerFrame", default_N=12, obs_len=800, num_frames=40))
    res = run_simulation(cfg)
    rep = summarize(res, cfg)
    row = csv_row("r0000", cfg, res, rep, 142000 / 74800)
    # the reference CLI's row for this run (kvweaver.cli._csv_row, captured once)
    assert row == ["r0000", "Unified", "CostModel", "12", "4", "10", "10", "1.000000", "OnePerFrame", "1", "42",
                   "133.689840", "133.689840", "160.427807", "3.000000", "0.000000", "3", "1.898396"]
    assert len(row) == len(CSV_COLUMNS)
    text = write_csv([row])
    assert text.splitlines()[0] == "# kvweaver-csv v1" and text.splitlines()[2] == ",".join(CSV_COLUMNS)


def test_extra_language_tasks_share_the_arrival():
    """Arrival.extra_tasks: one prefill, several language
    requests on the same prefix handle — batched together in the frame's decode."""
    from paper_2603_14371_b200 import (Arrival, KvManager, Observation, make_backend, BackendConfig,
                                       CostModelParams)
    from paper_2603_14371_b200.scheduler import run_frame_unified
    be = make_backend("CostModel", BackendConfig(), CostModelParams())
    mgr = KvManager()
    arr = [Arrival(0, Observation((1, 2, 3), 0), 4, extra_tasks=(6, 2))]
    res = run_frame_unified(0, arr, mgr, be, 2, 30.0)
    assert res.trace.batch_size_m == 3 and res.trace.prefill_count == 1
    states = [mgr.retrieve(r) for r in mgr.active_ids()]  # the 2-token task finished this frame
    assert sorted(s.max_len for s in states) == [4, 6] and all(len(s.tokens) == 2 for s in states)
    assert len(res.finished) == 1 and len(res.finished[0][1]) == 2
    # one action chunk per observation, recorded under every task's request id
    assert len(res.actions) == 3 and all(c is res.actions[0][1] for _, c in res.actions)
    import pytest
    with pytest.raises(ValueError):
        Arrival(0, Observation((1,), 0), 4, extra_tasks=(0,))


def test_extra_tasks_get_action_entries_and_complete():
    """Arrival.extra_tasks (several language tasks on one observation): every task's
    request id gets the observation's action chunk, so a frame loop can transcribe
    it when it completes (no orphaned request ids)."""
    from paper_2603_14371_b200 import Arrival, KvManager, Observation
    from paper_2603_14371_b200.backend import BackendConfig, CostModelParams, make_backend
    from paper_2603_14371_b200.scheduler import run_frame_unified
    be = make_backend("CostModel", BackendConfig(), CostModelParams())
    mgr = KvManager()
    res = run_frame_unified(0, [Arrival(0, Observation((1, 2, 3), 0), 2, extra_tasks=(5, 3))], mgr, be, 2, 30.0)
    rids = [rid for rid, _ in res.actions]
    assert sorted(rids) == [0, 1, 2]
    assert all(chunk == res.actions[0][1] for _, chunk in res.actions)
    pending = {rid for rid, _ in res.actions}
    pending -= {rid for rid, _ in res.finished}
    for t in range(1, 4):
        res = run_frame_unified(t, [], mgr, be, 2, 30.0)
        pending -= {rid for rid, _ in res.finished}
    assert not pending and not mgr.active_ids()


def test_deferred_action_chunk_behaves_as_action_chunk():
    """An overlapped frame's join yields DeferredActionChunk objects (pi05.py): the
    first read of .actions waits on the copy event, then converts and validates as
    ActionChunk does — same float64 values, equality, immutability and errors."""
    import torch
    from paper_2603_14371_b200.pi05 import DeferredActionChunk

    class Done:
        waited = 0

        def synchronize(self):
            Done.waited += 1

    host = torch.arange(2 * 5 * 3, dtype=torch.float32).reshape(2, 5, 3) / 7
    done = Done()
    d = DeferredActionChunk(host, 1, done)
    assert Done.waited == 0  # nothing is read until the chunk is used
    ref = ActionChunk(host[1].numpy().astype(np.float64))
    assert isinstance(d, ActionChunk)
    assert d == ref and ref == d and d.horizon == 5
    assert d.actions.dtype == np.float64 and not d.actions.flags.writeable
    assert Done.waited == 1
    _ = d.actions
    assert Done.waited == 1  # materialised once
    with pytest.raises(Exception):
        d.actions = None
    bad = host.clone()
    bad[0, 2, 1] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        _ = DeferredActionChunk(bad, 0, done).actions
