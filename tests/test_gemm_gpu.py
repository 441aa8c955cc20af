"""tcgen05 GEMM (csrc/gemm_sm100.cu) vs a plain PyTorch fp32 reference of the
same op on the same bf16 inputs.  Tolerance: fp32 accumulation in a
different order -> |err| <= 2e-3 * sqrt(K) * max|x||w| scale (stated per case)."""

import ctypes as C

import numpy as np
import pytest

from paper_2603_14371_b200 import _lib

pytestmark = pytest.mark.gpu


def run(w, x, mode=0, out=None, bias=None, res=None, splits=0):
    import torch
    n, k = w.shape
    t = x.shape[0]
    plan = np.zeros(6, np.int32)
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(splits),
              _lib.ptr_i32(plan))
    ws = torch.empty(max(1, int(plan[3]) * t * n), dtype=torch.float32, device="cuda")
    if out is None:
        if mode in (0, 2):
            out = torch.zeros(t, n, dtype=torch.float32, device="cuda")
        elif mode == 3:
            out = torch.zeros(t, n // 2, dtype=torch.bfloat16, device="cuda")
        else:
            out = torch.zeros(t, n, dtype=torch.bfloat16, device="cuda")
    _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
              C.c_int32(k), C.c_int32(t), C.c_int32(mode), C.c_void_p(out.data_ptr()),
              C.c_int32(out.shape[1]), C.c_void_p(bias.data_ptr() if bias is not None else None),
              C.c_void_p(res.data_ptr() if res is not None else None),
              C.c_int32(res.shape[1] if res is not None else 0), C.c_int32(splits),
              C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), _lib.stream_ptr())
    torch.cuda.synchronize()
    return out, plan


def rand(shape, seed, scale=1.0):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(shape, generator=g) * scale).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("n,k,t,splits", [
    (256, 128, 16, 1), (128, 64, 1, 1), (2560, 2048, 1, 0), (2048, 2048, 50, 0),
    (2048, 2048, 800, 0), (200, 136, 37, 1), (384, 512, 300, 3), (1152, 4304, 256, 0),
    (257152 // 64, 2048, 5, 0), (2048, 2048, 2400, 2), (1152, 4304, 2304, 2),
])
def test_gemm_matches_torch_fp32(n, k, t, splits):
    w = rand((n, k), 1, 0.05)
    x = rand((t, k), 2)
    out, plan = run(w, x, 0, splits=splits)
    ref = x.float() @ w.float().T
    tol = 2e-3 * np.sqrt(k) * 0.05 * 4
    err = (out - ref).abs().max().item()
    assert err < tol, (err, tol, plan.tolist())


def test_epilogues():
    import torch
    n, k, t = 512, 256, 40
    w = rand((n, k), 3, 0.05)
    x = rand((t, k), 4)
    bias = torch.linspace(-1, 1, n, device="cuda")
    acc = x.float() @ w.float().T
    for splits in (1, 4):
        out, _ = run(w, x, 1, splits=splits)
        torch.testing.assert_close(out.float(), acc, rtol=1e-2, atol=2e-2)
        base = torch.randn(t, n, device="cuda")
        out2 = base.clone()
        run(w, x, 2, out=out2, splits=splits)
        torch.testing.assert_close(out2, base + acc, rtol=1e-4, atol=2e-3)
        out3, _ = run(w, x, 3, splits=splits)
        g, u = acc[:, 0::2], acc[:, 1::2]
        gelu = 0.5 * g * (1 + torch.tanh(0.7978845608028654 * (g + 0.044715 * g ** 3)))
        torch.testing.assert_close(out3.float(), gelu * u, rtol=2e-2, atol=2e-2)
        out4, _ = run(w, x, 4, bias=bias, splits=splits)
        h = acc + bias
        torch.testing.assert_close(out4.float(), 0.5 * h * (1 + torch.tanh(
            0.7978845608028654 * (h + 0.044715 * h ** 3))), rtol=2e-2, atol=2e-2)
        res = torch.randn(t, n, device="cuda")
        out5, _ = run(w, x, 5, res=res, splits=splits)
        torch.testing.assert_close(out5.float(), acc + res, rtol=2e-2, atol=3e-2)


def test_split_k_is_deterministic_and_close_to_single():
    w = rand((1024, 2048), 5, 0.05)
    x = rand((8, 2048), 6)
    a, _ = run(w, x, 0, splits=8)
    b, _ = run(w, x, 0, splits=8)
    c, _ = run(w, x, 0, splits=1)
    assert (a == b).all()
    assert (a - c).abs().max().item() < 1e-3


@pytest.mark.parametrize("n,k,t,pad", [(4304, 256, 37, 0), (200, 136, 33, 0), (512, 128, 50, 3), (96, 64, 17, 1)])
def test_bf16_epilogues_ragged(n, k, t, pad):
    """bf16 outputs go through the per-warp smem transpose and 16-byte stores:
    ragged features (n % 32), ragged tokens (t % 16) and a row stride that is not
    a multiple of 8 (pad > 0: the scalar fall-back) against torch fp32."""
    import torch
    w = rand((n, k), 7, 0.05)
    x = rand((t, k), 8)
    bias = torch.linspace(-1, 1, n, device="cuda")
    acc = x.float() @ w.float().T
    out = torch.zeros(t, n + pad, dtype=torch.bfloat16, device="cuda")
    run(w, x, 1, out=out, splits=1)
    torch.testing.assert_close(out[:, :n].float(), acc, rtol=1e-2, atol=2e-2)
    assert (out[:, n:] == 0).all()
    out = torch.zeros(t, n + pad, dtype=torch.bfloat16, device="cuda")
    run(w, x, 4, out=out, bias=bias, splits=1)
    h = acc + bias
    torch.testing.assert_close(out[:, :n].float(), 0.5 * h * (1 + torch.tanh(
        0.7978845608028654 * (h + 0.044715 * h ** 3))), rtol=2e-2, atol=2e-2)
    if n % 2 == 0:
        out = torch.zeros(t, n // 2 + pad, dtype=torch.bfloat16, device="cuda")
        run(w, x, 3, out=out, splits=1)
        g, u = acc[:, 0::2], acc[:, 1::2]
        gelu = 0.5 * g * (1 + torch.tanh(0.7978845608028654 * (g + 0.044715 * g ** 3)))
        torch.testing.assert_close(out[:, :n // 2].float(), gelu * u, rtol=2e-2, atol=2e-2)
        assert (out[:, n // 2:] == 0).all()


@pytest.mark.parametrize("n,k,splits,mode", [(2560, 2048, 7, 1), (32768, 2048, 1, 3), (2048, 16384, 9, 0),
                                             (2048, 2048, 2, 2), (1024, 4096, 16, 0), (2560, 2048, 2, 1),
                                             (1152, 4304, 2, 2), (2048, 16384, 2, 0)])
def test_rows_independent_of_token_count(n, k, splits, mode):
    """Batch invariance of the GEMM: with the K partition fixed (the model's
    policy), a token row's output is bit-identical whether it is projected alone
    or inside 12, 64, 96, 400 or 2400 rows (different token tiles, 1- and 2-CTA
    kernels; at 2400 rows a split-2 partition runs both K halves in one CTA pair,
    summed in its epilogue instead of through fp32 partials and a reduce launch)."""
    import torch
    w = rand((n, k), 3, 0.02)
    xs = rand((2400, k), 4)
    base = None
    for t in (1, 12, 64, 96, 400, 2400):
        out, plan = run(w, xs[:t].contiguous(), mode, splits=splits)
        row = out[:1].clone()
        if base is None:
            base = row
        else:
            assert torch.equal(row, base), (t, plan.tolist(), (row.float() - base.float()).abs().max().item())
