"""One full-shape denoise through the persistent layer program inside
cudaProfilerStart/Stop (for `ncu --profile-from-start off -k regex:mk_kernel`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402


def main():
    os.environ.setdefault("OXY_MK", "1")
    cfg = Pi05Config()
    be = Pi05Backend(cfg, num_blocks=64)
    kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
    S = int(os.environ.get("S", "1"))
    for _ in range(3):
        be.action_denoise(kv, S)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    be.action_denoise(kv, S)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("probed")


if __name__ == "__main__":
    main()
