"""Per-event timeline of the skinny tcgen05 GEMM inside the denoise chain
(timing build: tools/prof_build.sh; OXY_LIB_VARIANT=aprof).  For weight tile 0 /
token tile 0 of the last launch with the given (n_out, k), prints each split
CTA's %globaltimer events in us relative to the earliest entry.
  python tools/gemm_prof.py N_OUT K      e.g. 8192 1024 (expert gate/up)"""
import ctypes as C
import os
import sys

os.environ.setdefault("OXY_LIB_VARIANT", "aprof")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images  # noqa: E402

EV = ["entry", "setup", "pre_issued", "prod_wait", "loads_issued", "mma_first", "mma_done", "epi_wait",
      "acc_ready", "epi_stored", "exit", "chunk0", "chunk1", "csk_sync", "csk_epi", "csk_norm",
      "full1", "full2", "full3", "-", "-", "-", "-", "-"]
n_out, k = int(sys.argv[1]), int(sys.argv[2])
be = Pi05Backend(Pi05Config(), num_blocks=64)
assert _lib.lib().oxy_debug_gemm_prof_select(n_out, k) == 0
kv = be.prefill(Pi05Observation(tuple(range(100, 132)), 0, synthetic_images(3, 5)))
for _ in range(4):
    be.denoise_many([kv], 10)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (32 * 24))()
assert _lib.lib().oxy_debug_gemm_prof(buf) == 0
a = np.array(buf, dtype=np.int64).reshape(32, 24)
rows = [i for i in range(32) if a[i, 0] > 0]
t0 = min(a[i, 0] for i in rows)
print(f"n_out {n_out} k {k}\nsplit " + " ".join(f"{e:>12s}" for e in EV))
for i in rows:
    print(f"{i:5d} " + " ".join(f"{(a[i, j] - t0) / 1e3:12.2f}" if a[i, j] >= t0 else f"{'-':>12s}"
                                for j in range(len(EV))))
if hasattr(_lib.lib(), "oxy_debug_gemm_prof2"):
    try:
        b2 = (C.c_ulonglong * (32 * 8))()
        if _lib.lib().oxy_debug_gemm_prof2(b2) == 0:
            a2 = np.array(b2, dtype=np.int64).reshape(32, 8)
            for i in rows[:2]:
                print("epi chunk0 events", [round((a2[i, j] - t0) / 1e3, 2) for j in range(3) if a2[i, j] > 0])
    except AttributeError:
        pass
