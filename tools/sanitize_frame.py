"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): TINY pi0.5 frames through the public API (prefill with a
camera, batched prefill, denoise on the expert lane overlapping a batched
decode, decode across a block boundary, copy-on-write forks), the F1 toy frame,
the paged decode attention in chunk and row modes, the tcgen05 prefix
attention with split merges (7 and 2 splits), the tcgen05 SigLIP attention and
the persistent 2-CTA GEMM with split K.  Run with OXY_GRAPHS=0 so every kernel launches
eagerly under the tool."""

import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_14371_b200 import _lib, Arrival, BackendConfig, BatchedState, KvManager, Observation  # noqa: E402
from paper_2603_14371_b200.pi05 import TINY, Pi05Backend, Pi05Observation, synthetic_images  # noqa: E402
from paper_2603_14371_b200.scheduler import run_frame_unified  # noqa: E402
from paper_2603_14371_b200.toy_b200 import ToyBackend  # noqa: E402


def pi05_frames():
    be = Pi05Backend(TINY, num_blocks=128)
    mgr = KvManager()
    for t in range(3):
        arr = [Arrival(t, Pi05Observation((5 + t, 17, 99, 3), t, synthetic_images(1, 11 + t)), 6, extra_tasks=(4,)),
               Arrival(t, Pi05Observation(tuple(range(40, 110)), t, None), 5)]
        run_frame_unified(t, arr, mgr, be, 3, 30.0)
    kv = be.prefill(Pi05Observation(tuple(range(2, 62)), 0, None))
    be.batched_language_decode(BatchedState((kv, kv), ((), ()), (False, False), (0, 1), (2, 9), (0, 0)), 8)
    be.recompute_logits([5, 6, 7, 1, 9])
    torch.cuda.synchronize()


def toy_frame():
    be = ToyBackend(BackendConfig(d_model=64, n_heads=2, vocab=128))
    mgr = KvManager()
    for t in range(2):
        run_frame_unified(t, [Arrival(t, Observation(tuple(range(3, 40)), t), 5)], mgr, be, 3, 30.0)
    torch.cuda.synchronize()


def decode_attention(rows, ctx):
    nb_row = -(-ctx // 64)
    nb = rows * nb_row + 1
    kp = torch.randn(nb, 64, 256, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, 64, 256, device="cuda", dtype=torch.bfloat16)
    bt = torch.randperm(nb, device="cuda")[: rows * nb_row].to(torch.int32).reshape(rows, nb_row).contiguous()
    pos = torch.full((rows,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, 2048, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    ws = torch.empty(rows * nb_row * 8 * 258, device="cuda", dtype=torch.float32)
    _lib.call("oxy_paged_decode_attention", C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
              C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()),
              C.c_int32(nb_row), C.c_void_p(pos.data_ptr()), C.c_int32(rows), C.c_int32(nb_row),
              C.c_void_p(ws.data_ptr()), _lib.stream_ptr())
    torch.cuda.synchronize()


def vit_attention(n_images=3, heads=16):
    qkv = torch.randn(n_images * 256, 3 * 72 * heads, device="cuda").to(torch.bfloat16)
    out = torch.empty(n_images * 256, 72 * heads, device="cuda", dtype=torch.bfloat16)
    _lib.call("oxy_vit_attention", C.c_void_p(qkv.data_ptr()), C.c_void_p(out.data_ptr()), C.c_int32(n_images),
              C.c_int32(heads), _lib.stream_ptr())
    torch.cuda.synchronize()


def prefix_attention(nq, nka, nkb, splits):
    nb = (nka + 63) // 64 + 2
    kp = torch.randn(nb, 64, 256, device="cuda").to(torch.bfloat16)
    vp = torch.randn(nb, 64, 256, device="cuda").to(torch.bfloat16)
    bt = torch.arange((nka + 63) // 64, device="cuda", dtype=torch.int32)
    q = torch.randn(nq, 256, device="cuda").to(torch.bfloat16)
    kd = torch.randn(max(nkb, 1), 256, device="cuda").to(torch.bfloat16)
    vd = torch.randn(max(nkb, 1), 256, device="cuda").to(torch.bfloat16)
    out = torch.empty(nq, 256, device="cuda", dtype=torch.bfloat16)
    rows = (nq + 127) // 128 * 128
    ws_o = torch.empty(splits * rows * 256, device="cuda")
    ws_ml = torch.empty(splits * rows * 2, device="cuda")
    _lib.call("oxy_prefix_attention", C.c_void_p(q.data_ptr()), C.c_void_p(out.data_ptr()),
              C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()),
              C.c_int32(nka), C.c_void_p(kd.data_ptr() if nkb else None), C.c_void_p(vd.data_ptr() if nkb else None),
              C.c_int32(nkb), C.c_int32(nq), C.c_int32(splits), C.c_void_p(ws_o.data_ptr()),
              C.c_void_p(ws_ml.data_ptr()), _lib.stream_ptr())
    torch.cuda.synchronize()


def wide_split_gemm(n=2560, k=2048, t=2400, mode=2, splits=2):
    """persistent 2-CTA kernel with split K: partials + the reduce kernel"""
    w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    x = torch.randn(t, k, device="cuda").to(torch.bfloat16)
    o = torch.zeros(t, n, device="cuda")
    ws = torch.empty(splits * t * n, device="cuda")
    _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(k),
              C.c_int32(t), C.c_int32(mode), C.c_void_p(o.data_ptr()), C.c_int32(n), None, None, C.c_int32(0),
              C.c_int32(splits), C.c_void_p(ws.data_ptr()), C.c_int64(ws.numel()), _lib.stream_ptr())
    torch.cuda.synchronize()


if __name__ == "__main__":
    pi05_frames()
    toy_frame()
    decode_attention(4, 700)   # chunk items + fold kernel
    decode_attention(48, 300)  # whole-row items
    vit_attention()             # tcgen05 SigLIP attention
    prefix_attention(400, 800, 50, 7)   # cluster merge, 7 splits (merge_rows<8>)
    prefix_attention(256, 800, 0, 2)    # cluster merge, 2 splits (merge_rows<2>)
    wide_split_gemm()           # wide kernel, split K -> partials + reduce kernel
    print("sanitize workload done")
