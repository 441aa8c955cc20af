"""Warm CUDA-event timing of the tcgen05 GEMM at the frame's shapes.
Usage: OXY_SPLITK=fixup|kernel OXY_PDL=0|1 OXY_GEMM_SMEM_KB=N python tools/gemm_bench.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402

SHAPES = [  # (name, n_out, k, t)
    ("dec qkv", 2560, 2048, 6), ("dec wo", 2048, 2048, 6), ("dec gu", 32768, 2048, 6),
    ("dec down", 2048, 16384, 6), ("dec lm", 257152, 2048, 6),
    ("dn qkv", 2560, 1024, 50), ("dn wo", 1024, 2048, 50), ("dn gu", 8192, 1024, 50),
    ("dn down", 1024, 4096, 50),
    ("pf qkv", 2560, 2048, 800), ("pf wo", 2048, 2048, 800), ("pf gu", 32768, 2048, 800),
    ("pf down", 2048, 16384, 800), ("vit fc1", 4304, 1152, 768), ("vit fc2", 1152, 4304, 768),
]


def main():
    st = torch.cuda.current_stream()
    tag = f"splitk={os.environ.get('OXY_SPLITK', 'kernel')} pdl={os.environ.get('OXY_PDL', '1')} smem={os.environ.get('OXY_GEMM_SMEM_KB', '200')}"
    print(tag)
    for name, n, k, t in SHAPES:
        w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
        x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
        o = torch.empty(t, n, device="cuda", dtype=torch.float32)
        plan = (C.c_int32 * 6)()
        _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
        ws = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
        args = (C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k),
                C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n), None, None,
                C.c_int32(0), C.c_int32(0), C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()),
                C.c_void_p(st.cuda_stream))
        for _ in range(3):
            _lib.call("oxy_gemm_bf16", *args)
        reps = 20
        # chain reps launches inside one CUDA graph-free burst; time on device
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            _lib.call("oxy_gemm_bf16", *args)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / reps * 1e3
        byts = n * k * 2
        fl = 2.0 * n * k * t
        print(f"{name:9s} n={n:6d} k={k:5d} t={t:3d} bn={plan[0]:3d} tiles={plan[1]}x{plan[2]} "
              f"splits={plan[3]:2d} st={plan[4]} {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s "
              f"{fl / us / 1e6:7.1f} TF/s")
        ref = x.float() @ w.float().T
        err = (o - ref).abs().max().item()
        assert err < 0.05, (name, err)


if __name__ == "__main__":
    main()
