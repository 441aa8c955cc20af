"""Prefill + one denoise at the full shape (for `ncu -k regex:<kernel> -s <n>`
captures of the denoise-path kernels; the prefill's launches come first)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402

be = Pi05Backend(Pi05Config(), num_blocks=64)
kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
be.action_denoise(kv, int(os.environ.get("S", "1")))
torch.cuda.synchronize()
print("probed")
