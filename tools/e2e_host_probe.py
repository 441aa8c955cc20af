"""Host-side time per frame of the end-to-end frame loop (numpy camera frames through
the public API): wall time per run_frame_unified call and inside the image upload,
against the GPU frame time (CUDA events) — where the host can leave the GPU idle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_14371_b200.kv_manager import KvManager  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config  # noqa: E402
from paper_2603_14371_b200.scheduler import run_frame_unified  # noqa: E402

cfg = Pi05Config()
be = Pi05Backend(cfg, num_blocks=352)
for device in (True, False):
    frames = bench.build_frames(cfg, [0], 28, 30, device=device)
    acc = {"img": 0.0}
    orig = be._images_device

    def timed_images(obs_list):
        t = time.perf_counter()
        r = orig(obs_list)
        acc["img"] += time.perf_counter() - t
        return r
    be._images_device = timed_images
    mgr = KvManager()
    for t in range(8):
        run_frame_unified(t, frames[t], mgr, be, 5, 30.0)
    torch.cuda.synchronize()
    acc["img"] = 0.0
    walls = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(8, 28):
        w = time.perf_counter()
        run_frame_unified(t, frames[t], mgr, be, 5, 30.0)
        walls.append(time.perf_counter() - w)
    e.record()
    torch.cuda.synchronize()
    be._images_device = orig
    print(f"{'device' if device else 'host'} frames: GPU {s.elapsed_time(e) / 20:.3f} ms/frame, host call "
          f"{1e3 * sum(walls) / 20:.3f} ms/frame (min {1e3 * min(walls):.3f}), image upload "
          f"{1e3 * acc['img'] / 20:.3f} ms/frame", flush=True)
