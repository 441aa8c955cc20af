import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2603_14371_b200 import _lib
st = torch.cuda.current_stream()
def bench(n, k, t, splits, mode, nbuf=40):
    ws_ = [torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(nbuf)]
    x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    plan = (C.c_int32 * 6)()
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(splits), plan)
    wsp = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
    def f(w):
        _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(mode), C.c_void_p(o.data_ptr()), C.c_int32(n // (2 if mode == 3 else 1)), None, None, C.c_int32(0), C.c_int32(splits), C.c_void_p(wsp.data_ptr()), C.c_int64(wsp.numel()), C.c_void_p(st.cuda_stream))
    for w in ws_: f(w)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(40): f(ws_[i % nbuf])
    e.record(); torch.cuda.synchronize()
    print(f"n={n} k={k} t={t} mode={mode} splits={plan[3]} {s.elapsed_time(e)/40*1e3:.1f} us", flush=True)
for mode in (0, 3, 4):
    for sp in (1, 2):
        bench(8192, 1024, 50, sp, mode)
