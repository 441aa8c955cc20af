"""N>1 host path on CPU: two gloo ranks each run their shard of independent
robot streams (cost backend, Uniform(r) arrivals) and reduce metrics exactly
like bench.py does on NCCL; the aggregate must equal the single-process run."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2603_14371_b200 import CostModelParams, SimConfig, WorkloadSpec, run_simulation
from paper_2603_14371_b200.sharding import reduce_metrics, streams_for_rank

TOTAL, FRAMES, H = 6, 12, 10


def _sim(r):
    cfg = SimConfig(variant="Unified", backend_kind="CostModel", cost_params=CostModelParams(),
                    workload=WorkloadSpec(pattern="Uniform", r=r, default_N=8, obs_len=50,
                                          num_frames=FRAMES), k=4)
    res = run_simulation(cfg)
    elapsed = sum(t.total_us for t in res.traces) / 1e6
    return elapsed, sum(t.actions_emitted for t in res.traces) // H, \
        sum(t.tokens_emitted for t in res.traces)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = streams_for_rank(TOTAL, world, rank)
    el, acts, toks = _sim(len(mine))
    out[rank] = reduce_metrics(el, acts, toks, len(mine), H)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_streams_partition():
    parts = [streams_for_rank(10, 4, r) for r in range(4)]
    assert sorted(s for p in parts for s in p) == list(range(10))
    assert parts[1] == [1, 5, 9]
    with pytest.raises(ValueError):
        streams_for_rank(4, 2, 2)


def test_two_rank_gloo_reduction_matches_single_process():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        got = dict(out)
    assert got[0] == got[1]                       # every rank sees the same aggregate
    el = max(_sim(len(streams_for_rank(TOTAL, world, r)))[0] for r in range(world))
    acts = sum(_sim(len(streams_for_rank(TOTAL, world, r)))[1] for r in range(world))
    assert got[0]["streams"] == TOTAL
    assert got[0]["actions"] == acts == TOTAL * FRAMES
    assert got[0]["action_hz"] == pytest.approx(H * acts / el)


def _bench_worker(rank, world, port, out):
    """bench.py's own end-of-run reduction (bench.aggregate -> sharding.reduce_metrics)."""
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r: 10 + r ms elapsed, 20 stream-frames, 100 * (r + 1) tokens, 2 streams
    out[rank] = bench.aggregate(world, 10.0 + rank, 20, 100 * (rank + 1), 2, device="cpu")
    dist.barrier()
    dist.destroy_process_group()


def test_bench_aggregate_over_two_gloo_ranks():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        got = dict(out)
    assert got[0] == got[1]
    g = got[0]
    assert g["elapsed_s"] == pytest.approx(0.011)          # max over ranks
    assert g["actions"] == 40 and g["tokens"] == 300 and g["streams"] == 4
    assert g["action_hz"] == pytest.approx(50 * 40 / 0.011)  # H = 50 per stream-frame
    assert g["tok_s_per_stream"] == pytest.approx(300 / 0.011 / 4)


def test_bench_spawn_line_and_core_shares():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    cmd = bench.spawn_command(["--gpus", "4", "--steps", "3"], 4, 29512)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]
    cores = list(range(16))
    shares = [bench.host_cores_for(r, 4, cores) for r in range(4)]
    assert [len(s) for s in shares] == [4] * 4
    assert sorted(c for s in shares for c in s) == cores
    a = bench.args_parse(["--gpus", "8"])
    assert a.total_streams == 64   # configs[4] default for N > 1
    assert bench.args_parse([]).total_streams == 0
