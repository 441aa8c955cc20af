"""Full-shape A/B of the denoise paths: persistent layer program (OXY_MK=1)
vs the multi-kernel CUDA-graph path (OXY_MK=0) on the same prefix, plus a
CUDA-event timing of each.  Both are bf16 tcgen05 paths of the same math, so
they agree to bf16 rounding (different split-K / norm reduction trees)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def run(mk: str, S: int, reps: int):
    os.environ["OXY_MK"] = mk
    from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images
    cfg = Pi05Config()
    be = Pi05Backend(cfg, num_blocks=64)
    obs = Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5))
    kv = be.prefill(obs)
    acts = [be.action_denoise(kv, S).actions for _ in range(3)]  # eager, capture, replay
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        be.action_denoise(kv, S)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    del kv, be
    torch.cuda.empty_cache()
    return acts, ms


def main():
    S = int(os.environ.get("S", "10"))
    t0 = time.time()
    a1, ms1 = run("1", S, 10)
    print(f"mk: {ms1:.3f} ms/denoise  replay-identical={all(np.array_equal(a1[0], x) for x in a1)}", flush=True)
    a0, ms0 = run("0", S, 10)
    print(f"multi-kernel: {ms0:.3f} ms/denoise", flush=True)
    d = np.abs(a1[0] - a0[0]).max() / (np.abs(a0[0]).max() + 1e-9)
    print(f"max rel diff mk vs multi-kernel: {d:.3e}  (|a|max {np.abs(a0[0]).max():.3f})  {time.time() - t0:.0f}s")
    assert d < 3e-2


if __name__ == "__main__":
    main()
