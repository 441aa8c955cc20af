"""Host-side profile of the e2e frame loop (bench.py's e2e leg: numpy camera
frames through run_frame_unified).  Prints device-frame vs host-frame ms per
frame and the top cProfile entries of the host-frame loop, so host work that
sits on the critical path shows up.  Usage (GPU box): python tools/e2e_profile.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14371_b200.kv_manager import KvManager  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config  # noqa: E402
from paper_2603_14371_b200.scheduler import run_frame_unified  # noqa: E402


def loop(backend, frames, warm, k=5):
    mgr = KvManager()
    for t in range(warm):
        run_frame_unified(t, frames[t], mgr, backend, k, 30.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(warm, len(frames)):
        run_frame_unified(t, frames[t], mgr, backend, k, 30.0)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / (len(frames) - warm)


def main():
    cfg = Pi05Config()
    n, warm = 28, 8
    backend = Pi05Backend(cfg, num_blocks=512, measure=False)
    dev = bench.build_frames(cfg, [0], n, 30, device=True)
    host = bench.build_frames(cfg, [0], n, 30, device=False)
    print(f"device frames: {loop(backend, dev, warm):.3f} ms/frame")
    print(f"host frames:   {loop(backend, host, warm):.3f} ms/frame")
    pr = cProfile.Profile()
    mgr = KvManager()
    for t in range(warm):
        run_frame_unified(t, host[t], mgr, backend, 5, 30.0)
    torch.cuda.synchronize()
    pr.enable()
    for t in range(warm, n):
        run_frame_unified(t, host[t], mgr, backend, 5, 30.0)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
