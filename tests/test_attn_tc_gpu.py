"""The tcgen05 flash attention (csrc/attn_tc.cu) under every key-split regime:
one split per tile .. one split for all tiles, with paged + dense key tiles in
one CTA and O rescales, re-running the oracle parity tests of
tests/test_pi05_gpu.py in a fresh process per setting (the split knob is read
at model creation).  A timeout turns a pipeline deadlock into a failure."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tps,cmerge", [("1", "16"), ("2", "16"), ("3", "16"), ("7", "16"), ("1", "0"),
                                        ("64", "16")])
def test_attention_splits_match_oracle(tps, cmerge):
    """tps = key tiles per split for the prefill and the expert suffix (1: one split
    per tile .. 64: one split); cmerge 16: splits <= 16 merge over DSMEM inside the
    kernel; 0: workspace + fa_merge."""
    env = dict(os.environ, OXY_ATTN_TC="1", OXY_ATTN_TPS=f"{tps},{tps}", OXY_ATTN_CMERGE=cmerge)
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", os.path.join(ROOT, "tests", "test_pi05_gpu.py"),
           "-k", "prefill_kv or action_denoise or decode_logits or batch_invariant or graph_replay"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


@pytest.mark.parametrize("nq,nka,nkb,splits", [
    (64, 800, 0, 2), (400, 800, 50, 14), (400, 800, 50, 1), (1000, 100, 37, 3), (8, 64, 0, 1),
    (6400, 800, 0, 2), (130, 0, 77, 2), (256, 2000, 0, 32), (400, 800, 50, 12), (400, 800, 300, 16),
    (400, 1100, 0, 17)])
def test_prefix_attention_matches_torch(nq, nka, nkb, splits):
    """oxy_prefix_attention (tcgen05, paged + dense keys, split merge) against a
    torch fp32 softmax attention on the same bf16 inputs.  Tolerance: P is
    rounded to bf16 before P.V and the output is bf16 -> 2e-2 of max|V|."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(nq + nka + nkb)
    nb = max(1, (nka + 63) // 64) + 3
    kp = (torch.randn(nb, 64, 256, generator=g)).to(torch.bfloat16).cuda()
    vp = (torch.randn(nb, 64, 256, generator=g)).to(torch.bfloat16).cuda()
    perm = torch.randperm(nb, generator=g)[: max(1, (nka + 63) // 64)].to(torch.int32).cuda()
    q = (torch.randn(nq, 256, generator=g) * 2).to(torch.bfloat16).cuda()
    kd = torch.randn(max(nkb, 1), 256, generator=g).to(torch.bfloat16).cuda()
    vd = torch.randn(max(nkb, 1), 256, generator=g).to(torch.bfloat16).cuda()
    out = torch.zeros(nq, 256, dtype=torch.bfloat16, device="cuda")
    rows = (nq + 127) // 128 * 128  # (splits <= 16 merge in-kernel and leave the workspace untouched)
    ws_o = torch.empty(splits * rows * 256, device="cuda")
    ws_ml = torch.empty(splits * rows * 2, device="cuda")
    _lib.call("oxy_prefix_attention", C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
              C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(perm.data_ptr()),
              C.c_int32(nka), C.c_void_p(kd.data_ptr() if nkb else None), C.c_void_p(vd.data_ptr() if nkb else None),
              C.c_int32(nkb), C.c_int32(nq), C.c_int32(splits), C.c_void_p(ws_o.data_ptr()),
              C.c_void_p(ws_ml.data_ptr()), _lib.stream_ptr())
    torch.cuda.synchronize()
    keys = kp[perm.long()].reshape(-1, 256)[:nka].float()
    vals = vp[perm.long()].reshape(-1, 256)[:nka].float()
    if nkb:
        keys = torch.cat([keys, kd[:nkb].float()])
        vals = torch.cat([vals, vd[:nkb].float()])
    ref = torch.softmax(q.float() @ keys.T / 16.0, dim=-1) @ vals
    err = (out.float() - ref).abs().max().item()
    assert err < 2e-2 * vals.abs().max().item(), err


def test_prefix_attention_workspace_merge():
    """The same direct shapes with the in-kernel cluster merge off (workspace + fa_merge)."""
    env = dict(os.environ, OXY_ATTN_CMERGE="0")
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", os.path.abspath(__file__),
           "-k", "test_prefix_attention_matches_torch"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


@pytest.mark.parametrize("n_images,heads", [(1, 16), (3, 16), (2, 2), (5, 3)])
def test_vit_attention_matches_torch(n_images, heads):
    """oxy_vit_attention (tcgen05 SigLIP attention: head dim 72 run as K = 80 with Q
    zero-padded, all 256 keys per CTA) against torch fp32 softmax attention on the
    same bf16 fused qkv rows.  Tolerance: P and the output are bf16 -> 2e-2 of max|V|.
    The next head's dims ride along in the second 64-dim TMA box of every head, so
    a leak of them into S or O would show."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    D = 72 * heads
    g = torch.Generator(device="cpu").manual_seed(n_images * 100 + heads)
    qkv = torch.randn(n_images * 256, 3 * D, generator=g) * 1.5
    out = torch.zeros(n_images * 256, D, dtype=torch.bfloat16, device="cuda")
    qkv_b = qkv.to(torch.bfloat16)
    dev = qkv_b.cuda()
    _lib.call("oxy_vit_attention", C.c_void_p(dev.data_ptr()), C.c_void_p(out.data_ptr()), C.c_int32(n_images),
              C.c_int32(heads), _lib.stream_ptr())
    torch.cuda.synchronize()
    x = qkv_b.float().reshape(n_images, 256, 3, heads, 72)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [img, head, tok, 72]
    ref = torch.softmax(q @ k.transpose(-1, -2) / 72 ** 0.5, dim=-1) @ v
    ref = ref.permute(0, 2, 1, 3).reshape(n_images * 256, D)
    err = (out.float().cpu() - ref).abs().max().item()
    assert err < 2e-2 * v.abs().max().item(), err
