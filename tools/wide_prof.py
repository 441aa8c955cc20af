"""Tile timeline of the persistent wide GEMM (timing build: tools/prof_build.sh;
OXY_LIB_VARIANT=aprof).  Runs one standalone launch of (n_out, k, T, mode) and prints,
for CTAs 0..3 and each of their tiles, when the MMA warp started the tile
(accumulator free), issued its last k-block, and when epilogue warp 2 saw the
accumulator and finished — in us from the earliest kernel entry.
    python tools/wide_prof.py [N_OUT K T MODE]      (default: prefill gate/up 32768 2048 800 3)"""
import ctypes as C
import os
import sys

os.environ.setdefault("OXY_LIB_VARIANT", "aprof")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402

n, k, t, mode = [int(a) for a in sys.argv[1:5]] if len(sys.argv) >= 5 else (32768, 2048, 800, 3)
st = torch.cuda.current_stream()
w = (torch.randn(n, k) * 0.02).to(torch.bfloat16).cuda()
x = torch.randn(t, k).to(torch.bfloat16).cuda()
cols = n // 2 if mode == 3 else n
o = torch.zeros(t, cols, device="cuda", dtype=torch.float32 if mode == 0 else torch.bfloat16)
plan = (C.c_int32 * 6)()
_lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
ws = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
assert _lib.lib().oxy_debug_gemm_prof_select(n, k) == 0
for _ in range(4):
    _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k),
              C.c_int32(t), C.c_int32(mode), C.c_void_p(o.data_ptr()), C.c_int32(cols), None, None, C.c_int32(0),
              C.c_int32(0), C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), C.c_void_p(st.cuda_stream))
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4 * 17 * 6))()
assert _lib.lib().oxy_debug_wide_prof(buf) == 0
a = np.array(buf, dtype=np.int64).reshape(4, 17, 6)
t0 = a[:, 16, 0][a[:, 16, 0] > 0].min()
f = lambda v: f"{(v - t0) / 1e3:8.2f}" if v >= t0 else f"{'-':>8s}"
print("(clock: clock64 / globaltimer between the MMA warp's tile start and last issue)")
print(f"n_out {n} k {k} T {t} mode {mode} plan {list(plan)}  env {os.environ.get('OXY_GEMM_WIDE_DIAG', '')}")
for c in range(4):
    print(f"cta {c}: entry {f(a[c, 16, 0])} setup {f(a[c, 16, 1])} exit {f(a[c, 16, 2])}")
    for lt in range(16):
        if a[c, lt, :4].max() >= t0:
            mhz = (a[c, lt, 5] - a[c, lt, 4]) / max(1, a[c, lt, 1] - a[c, lt, 0]) * 1e3 if a[c, lt, 0] >= t0 else 0
            print(f"   tile {lt:2d}: mma start {f(a[c, lt, 0])} issued {f(a[c, lt, 1])}  epi acc {f(a[c, lt, 2])} "
                  f"done {f(a[c, lt, 3])}  SM clock over the mainloop {mhz:6.0f} MHz")
