"""Run one hot kernel a few times at a frame shape (for `ncu --set full`).

    python tools/kernel_probe.py gemm 32768 2048 800      # n_out k tokens
    python tools/kernel_probe.py decode_attention 64 1024 # rows ctx
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14371_b200 import _lib  # noqa: E402


def gemm(n, k, t, reps=5):
    st = torch.cuda.current_stream()
    w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
    x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    plan = (C.c_int32 * 6)()
    _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
    ws = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
    for _ in range(reps):
        _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
                  C.c_int32(k), C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n),
                  None, None, C.c_int32(0), C.c_int32(0), C.c_void_p(ws.data_ptr()),
                  C.c_int64(ws.numel()), C.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()


def decode_attention(rows, ctx, reps=5):
    st = torch.cuda.current_stream()
    blk = 64
    nb = rows * ctx // blk
    kp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    bt = torch.randperm(nb, device="cuda").to(torch.int32).reshape(rows, ctx // blk).contiguous()
    pos = torch.full((rows,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, 2048, device="cuda", dtype=torch.bfloat16)
    ob = torch.empty_like(q)
    ws = torch.empty(rows * (ctx // blk) * 8 * 258, device="cuda", dtype=torch.float32)
    for _ in range(reps):
        _lib.call("oxy_paged_decode_attention", C.c_void_p(q.data_ptr()), C.c_void_p(ob.data_ptr()),
                  C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()),
                  C.c_int32(ctx // blk), C.c_void_p(pos.data_ptr()), C.c_int32(rows),
                  C.c_int32(ctx // blk), C.c_void_p(ws.data_ptr()), C.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()


if __name__ == "__main__":
    kind = sys.argv[1]
    args = [int(a) for a in sys.argv[2:]]
    {"gemm": gemm, "decode_attention": decode_attention}[kind](*args)
    print("ok", kind, args)
