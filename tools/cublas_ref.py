"""cuBLAS (torch.matmul, bf16) on the frame's GEMM shapes: the library
yardstick for tools/gemm_bench.py (weights [n, k], activations [t, k])."""
import torch

SHAPES = [("pf qkv", 2560, 2048, 800), ("pf wo", 2048, 2048, 800), ("pf gu", 32768, 2048, 800),
          ("pf down", 2048, 16384, 800), ("vit qkv", 3456, 1152, 768), ("vit wo", 1152, 1152, 768),
          ("vit fc1", 4304, 1152, 768), ("vit fc2", 1152, 4304, 768), ("dn qkv", 2560, 1024, 50),
          ("dn gu", 8192, 1024, 50), ("dn down", 1024, 4096, 50), ("dec gu", 32768, 2048, 6),
          ("dec lm", 257152, 2048, 6)]
for name, n, k, t in SHAPES:
    w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        y = x @ w.T
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        y = x @ w.T
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 20 * 1e3
    print(f"{name:8s} n={n:6d} k={k:5d} t={t:3d} cublas {us:8.1f} us {2*n*k*t/us/1e6:7.1f} TF/s {n*k*2/us/1e3:6.0f} GB/s")
