"""One ViT-shaped prefill GEMM through the C ABI (for ncu): qkv 3456x1152 or fc1
4304x1152 at T = 768 tokens (3 cameras x 256 patches), warm."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402

n, k, t = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (3456, 1152, 768)))
st = torch.cuda.current_stream()
w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
o = torch.empty(t, n, device="cuda", dtype=torch.bfloat16)
ws = torch.empty(4 * t * n, device="cuda", dtype=torch.float32)
args = (C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(1),
        C.c_void_p(o.data_ptr()), C.c_int32(n), None, None, C.c_int32(0), C.c_int32(0),
        C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), C.c_void_p(st.cuda_stream))
plan = (C.c_int32 * 6)()
_lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
print("plan bn,n_tiles,m_tiles,splits,stages,kb", list(plan))
for _ in range(5):
    _lib.call("oxy_gemm_bf16", *args)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    _lib.call("oxy_gemm_bf16", *args)
e.record()
torch.cuda.synchronize()
us = s.elapsed_time(e) / 20 * 1e3
print(f"{n}x{k} T={t}: {us:.2f} us, {2 * n * k * t / us / 1e6:.1f} TFLOP/s")
