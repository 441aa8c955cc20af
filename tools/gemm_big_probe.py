"""Big-T prefill GEMMs (multi-stream frames: T = streams x 800): ours vs cuBLAS."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14371_b200 import _lib
st = torch.cuda.current_stream()
for name, n, k, t in [("gu", 32768, 2048, 6400), ("down", 2048, 16384, 6400), ("qkv", 2560, 2048, 6400),
                      ("gu", 32768, 2048, 800), ("down", 2048, 16384, 800)]:
    w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
    x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    plan = (C.c_int32 * 6)()
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
    ws = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
    f = lambda: _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n), None, None, C.c_int32(0), C.c_int32(0), C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), C.c_void_p(st.cuda_stream))
    g = lambda: torch.matmul(x, w.T)
    for fn, lab in ((f, "ours"), (g, "cublas")):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): fn()
        e.record(); torch.cuda.synchronize()
        us = s.elapsed_time(e) / 10 * 1e3
        print(f"{name:5s} n={n} k={k} t={t} {lab:6s} {us:8.1f} us {2*n*k*t/us/1e6:7.1f} TF/s plan={list(plan)}", flush=True)
