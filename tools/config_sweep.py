"""BASELINE.json configs[2..4] on one B200 (the headline configs[1] is bench.py):

  multitask  configs[2]: unified frames, cross-frame continuously batched language
             requests, budget N x tokens-per-frame k sweep
  variants   configs[3]: Unified vs SharedNoBatch vs IsolatedSequential frames on
             the same inputs (kvweaver/scheduler.py:123, 194, 229)
  streams    configs[4]: r lock-stepped robot streams per GPU (64 streams over
             G = 2/4/8 GPUs -> r = 32/16/8; r = 1 is configs[1])

Prints one JSON line per point.  Timing: CUDA events around the steady frames
(after warm-up), clocks not sampled (bench.py does that for the headline).

  tasks      SURVEY.md §8f rank 4: 1 / 2 / 3 language tasks (memory, narration, ...)
             on each observation's shared prefix (Arrival.extra_tasks)

    python tools/config_sweep.py multitask|tasks|variants|streams|all
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14371_b200.kv_manager import KvManager  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config  # noqa: E402
from paper_2603_14371_b200.scheduler import (run_frame_isolated_sequential,  # noqa: E402
                                             run_frame_shared_no_batch, run_frame_unified)

H = 50


def run(backend, frames, warm, k, variant="Unified"):
    mgr = KvManager()
    rid = [0]

    def frame(t):
        arr = frames[t]
        if variant == "Unified":
            return run_frame_unified(t, arr, mgr, backend, k, 30.0)
        if variant == "SharedNoBatch":
            return run_frame_shared_no_batch(t, arr, mgr, backend, 30.0)
        res = run_frame_isolated_sequential(t, arr, backend, 30.0, rid[0])
        rid[0] += len(arr)
        return res

    for t in range(warm):
        frame(t)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    traces = [frame(t).trace for t in range(warm, len(frames))]
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / (len(frames) - warm)
    return ms, traces


def point(name, backend, cfg, streams, budget, k, steps, warm, variant="Unified", extra_tasks=0):
    frames = bench.build_frames(cfg, list(range(streams)), warm + steps, budget, device=True)
    if extra_tasks:  # memory + narration style: more language tasks on each observation's prefix
        import dataclasses
        frames = [[dataclasses.replace(a, extra_tasks=(budget,) * extra_tasks) for a in f] for f in frames]
    ms, traces = run(backend, frames, warm, k, variant)
    toks = sum(t.tokens_emitted for t in traces)
    line = {"sweep": name, "variant": variant, "streams_per_gpu": streams, "budget_N": budget, "k": k,
            "language_tasks_per_observation": 1 + extra_tasks,
            "frame_ms": round(ms, 3), "action_hz_per_stream_H50": round(H * 1e3 / ms, 1),
            "action_hz_per_stream_H10": round(10 * 1e3 / ms, 1),
            "action_hz_aggregate_H50": round(H * streams * 1e3 / ms, 1),
            "lang_tok_s_per_stream": round(toks / (ms * steps / 1e3) / streams, 1),
            "steady_batch": statistics.mean(t.batch_size_m for t in traces)}
    print(json.dumps(line), flush=True)
    return line


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    cfg = Pi05Config()
    if what in ("multitask", "all"):
        be = Pi05Backend(cfg, num_blocks=256 + 64 * 8)
        for budget, k in ((16, 1), (16, 5), (30, 1), (30, 5), (30, 10), (60, 5), (60, 10)):
            warm = max(4, -(-budget // k) + 2)
            point("multitask", be, cfg, 1, budget, k, 10, warm)
        del be
        torch.cuda.empty_cache()
    if what in ("tasks", "all"):  # several language tasks share one prefix
        be = Pi05Backend(cfg, num_blocks=1024)
        for extra in (0, 1, 2):
            point("tasks", be, cfg, 1, 30, 5, 8, 10, extra_tasks=extra)
        del be
        torch.cuda.empty_cache()
    if what in ("variants", "all"):
        be = Pi05Backend(cfg, num_blocks=512)
        for variant in ("Unified", "SharedNoBatch", "IsolatedSequential"):
            point("variants", be, cfg, 1, 30, 5, 6, 8, variant)
        del be
        torch.cuda.empty_cache()
    if what in ("streams", "all"):
        for r in (1, 8, 16, 32):
            be = Pi05Backend(cfg, num_blocks=256 + r * 8 * 14)
            point("streams", be, cfg, r, 30, 5, 5, 8)
            del be
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
