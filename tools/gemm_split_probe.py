"""Split-K sweep of the one-tile-per-CTA GEMM at the skinny frame shapes
(GEMM + its split-K reduce kernel, 40 distinct weight buffers so weights
stream from HBM).  Used to pick the skinny split policy."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2603_14371_b200 import _lib
st = torch.cuda.current_stream()
def bench(n, k, t, splits, nbuf):
    ws_ = [torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(nbuf)]
    x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    plan = (C.c_int32 * 6)()
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(splits), plan)
    wsp = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
    def f(w):
        _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n), None, None, C.c_int32(0), C.c_int32(splits), C.c_void_p(wsp.data_ptr()), C.c_int64(wsp.numel()), C.c_void_p(st.cuda_stream))
    for w in ws_: f(w)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 40
    s.record()
    for i in range(reps): f(ws_[i % nbuf])
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) / reps * 1e3
    print(f"n={n} k={k} t={t} splits={plan[3]} bn={plan[0]} nbuf={nbuf} {us:.1f} us  {n*k*2/us/1e3:.0f} GB/s", flush=True)
import sys as _s
CASES = [(2560, 1024, 50), (8192, 1024, 50), (1024, 4096, 50), (1024, 2048, 50), (32, 1024, 50),
         (2560, 2048, 6), (2048, 2048, 6), (2048, 16384, 6), (32768, 2048, 6)]
for n, k, t in CASES:
    for sp in (1, 2, 4, 8, 16):
        if sp <= (k + 63) // 64:
            bench(n, k, t, sp, 40)
