"""Paged decode attention (oxy_paged_decode_attention) at several rows x ctx
shapes: L2-flushed per-launch CUDA-event time, achieved HBM GB/s on the
algorithmic bytes (K + V of every row's context + q + out) and the fraction of
the measured HBM peak.  Prints one JSON line."""

import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_14371_b200 import _lib  # noqa: E402


def run(rows, ctx, timer, hbm):
    blk = 64
    mb = -(-ctx // blk)
    nb = rows * mb
    kp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    bt = torch.randperm(nb, device="cuda").to(torch.int32).reshape(rows, mb).contiguous()
    pos = torch.full((rows,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, 2048, device="cuda", dtype=torch.bfloat16)
    ob = torch.empty_like(q)
    wsd = torch.empty(rows * mb * 8 * 258, device="cuda", dtype=torch.float32)
    st = torch.cuda.current_stream()
    args = (C.c_void_p(q.data_ptr()), C.c_void_p(ob.data_ptr()), C.c_void_p(kp.data_ptr()),
            C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()), C.c_int32(mb),
            C.c_void_p(pos.data_ptr()), C.c_int32(rows), C.c_int32(mb), C.c_void_p(wsd.data_ptr()),
            C.c_void_p(st.cuda_stream))
    fn = lambda: _lib.call("oxy_paged_decode_attention", *args)  # noqa: E731
    sec = timer(fn, n=20)
    byts = rows * ctx * 256 * 2 * 2 + rows * 2048 * 2 * 2
    return {"rows": rows, "ctx": ctx, "mb": byts / 1e6, "us": sec * 1e6, "gbs": byts / sec / 1e9,
            "frac": byts / sec / 1e9 / hbm}


def main():
    hbm = bench.peaks()[0]
    timer = bench.ColdTimer()
    shapes = [(256, 1024), (512, 1024), (128, 2048), (64, 1024), (6, 832), (32, 832), (1, 8192)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
    print(json.dumps([run(r, c, timer, hbm) for r, c in shapes]))


if __name__ == "__main__":
    main()
