"""Run warm-up frames, then ONE steady frame inside cudaProfilerStart/Stop so
`ncu --profile-from-start off` sees exactly one frame's kernels.

    OXY_GREEN=0 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/frame_launches.csv python tools/profile_frame.py
    python tools/summarize_launches.py gpurun_out/frame_launches.csv

OXY_GREEN=0: cudaProfilerStart scopes the primary context, and the overlapped
denoise / decode otherwise run in their green-context SM partitions (the launch
list is serialised under ncu either way).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14371_b200.kv_manager import KvManager  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config  # noqa: E402
from paper_2603_14371_b200.scheduler import run_frame_unified  # noqa: E402


def main():
    streams = int(os.environ.get("STREAMS", "1"))
    warm = int(os.environ.get("WARM", "8"))
    cfg = Pi05Config()
    be = Pi05Backend(cfg, num_blocks=256 + streams * 64)
    frames = bench.build_frames(cfg, list(range(streams)), warm + 1, 30, device=True)
    mgr = KvManager()
    for t in range(warm):
        run_frame_unified(t, frames[t], mgr, be, 5, 30.0)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    run_frame_unified(warm, frames[warm], mgr, be, 5, 30.0)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one frame")


if __name__ == "__main__":
    main()
