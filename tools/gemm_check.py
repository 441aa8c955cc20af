"""Numerics check of the tcgen05 GEMM under the current OXY_GEMM_* knobs
(run in a fresh process per knob setting: the knobs are read once).

    OXY_GEMM_WIDE=2 OXY_GEMM_WIDE_BN=96 python tools/gemm_check.py

Every shape x epilogue mode is compared with a plain PyTorch fp32 reference
of the same op on the same bf16 inputs (tolerances as in tests/test_gemm_gpu.py)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402

SHAPES = [(256, 128, 80), (384, 512, 300), (2560, 2048, 800), (200, 136, 97), (1152, 4304, 256),
          (4304, 1152, 768), (512, 4096, 130)]


def run(w, x, mode, out, bias=None, res=None):
    n, k = w.shape
    t = x.shape[0]
    plan = (C.c_int32 * 6)()
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
    ws = torch.empty(max(1, plan[3] * t * n), dtype=torch.float32, device="cuda")
    _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k),
              C.c_int32(t), C.c_int32(mode), C.c_void_p(out.data_ptr()), C.c_int32(out.shape[1]),
              C.c_void_p(bias.data_ptr() if bias is not None else None),
              C.c_void_p(res.data_ptr() if res is not None else None), C.c_int32(res.shape[1] if res is not None else 0),
              C.c_int32(0), C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), _lib.stream_ptr())
    torch.cuda.synchronize()
    return list(plan)


def main():
    g = torch.Generator(device="cpu").manual_seed(0)
    for n, k, t in SHAPES:
        w = (torch.randn(n, k, generator=g) * 0.05).to(torch.bfloat16).cuda()
        x = torch.randn(t, k, generator=g).to(torch.bfloat16).cuda()
        acc = x.float() @ w.float().T
        tol = 2e-3 * k ** 0.5 * 0.05 * 4
        o0 = torch.zeros(t, n, device="cuda")
        plan = run(w, x, 0, o0)
        e0 = (o0 - acc).abs().max().item()
        base = torch.randn(t, n, device="cuda")
        o2 = base.clone()
        run(w, x, 2, o2)
        e2 = (o2 - base - acc).abs().max().item()
        o3 = torch.zeros(t, n // 2, dtype=torch.bfloat16, device="cuda")
        run(w, x, 3, o3)
        gg, u = acc[:, 0::2], acc[:, 1::2]
        ref3 = 0.5 * gg * (1 + torch.tanh(0.7978845608028654 * (gg + 0.044715 * gg ** 3))) * u
        e3 = ((o3.float() - ref3).abs() / (ref3.abs() + 1.0)).max().item()
        o0b = torch.zeros(t, n, device="cuda")
        run(w, x, 0, o0b)
        det = bool((o0 == o0b).all())
        ok = e0 < tol and e2 < tol + 1e-3 and e3 < 3e-2 and det
        print(f"n={n:5d} k={k:5d} t={t:4d} plan={plan} err f32={e0:.2e} add={e2:.2e} geglu={e3:.2e} "
              f"det={det} tol={tol:.2e} {'OK' if ok else 'FAIL'}", flush=True)
        assert ok


if __name__ == "__main__":
    main()
    print("gemm_check passed")
