"""Per-event timeline of the tcgen05 attention kernel inside the denoise chain
(needs the timing build: tools/prof_build.sh, OXY_LIB_VARIANT=aprof).
Prints, for query tile 0 of the LAST attention launch, each split CTA's
%globaltimer events in us relative to the earliest kernel entry.
  SKIP=<OXY_DBG_SKIP mask> for chain variants (57: attention kernels only)."""
import ctypes as C
import os
import sys

os.environ.setdefault("OXY_LIB_VARIANT", "aprof")
if os.environ.get("SKIP"):
    os.environ["OXY_DBG_SKIP"] = os.environ["SKIP"]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402

EV = ["entry", "trigger", "prod_wait", "q_landed", "smax_wait", "s0_ready", "p_last", "o_done", "staged",
      "tma_done", "syncthr", "cl_sync1", "merged", "cl_sync2", "s0_max", "exp_done", "s1_ready", "s1_max",
      "exp1_done", "-", "p2", "p3", "p4", "p5"]
be = Pi05Backend(Pi05Config(), num_blocks=64)
kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
for _ in range(4):
    if os.environ.get("PREFILL"):  # the last launch = the last Gemma layer's prefix attention
        del kv
        kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
        continue
    try:
        be.denoise_many([kv], 10)
    except ValueError:
        pass
torch.cuda.synchronize()
buf = (C.c_ulonglong * (32 * 24))()
assert _lib.lib().oxy_debug_attn_prof(buf) == 0
a = np.array(buf, dtype=np.int64).reshape(32, 24)
rows = [i for i in range(32) if a[i, 0] > 0]
t0 = min(a[i, 0] for i in rows)
print("split " + " ".join(f"{e:>9s}" for e in EV))
for i in rows:
    print(f"{i:5d} " + " ".join(f"{(a[i, j] - t0) / 1e3:9.2f}" if a[i, j] >= t0 else f"{'-':>9s}"
                                for j in range(len(EV))))
