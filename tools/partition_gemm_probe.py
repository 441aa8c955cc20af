"""Decode / denoise projections timed on an SM partition (green context) vs all SMs:
each projection at its frame plan (policy split-K + reduce), 20 back-to-back launches
on a stream of a green context with N SMs, weights larger than L2 rotated so they
stream from HBM.  Prints GB/s of weight bytes per shape.
    python tools/partition_gemm_probe.py [N_SMS ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import cuda.bindings.driver as drv  # noqa: E402

import bench  # noqa: E402
from paper_2603_14371_b200 import _lib  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Config  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


def green_stream(n_sms):
    torch.cuda.init()
    dev = ck(drv.cuDeviceGet(0))
    res = ck(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    out = drv.cuDevSmResourceSplitByCount(1, res, 0, n_sms)
    groups, _, rest = out[1], out[2], out[3]
    desc = ck(drv.cuDevResourceGenerateDesc([groups[0]], 1))
    g = ck(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    s = ck(drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    return int(s), groups[0].sm.smCount, g


def main():
    cfg = Pi05Config()
    llm, exp, _ = bench.projections(cfg)
    shapes = [("dec.qkv", *llm[0], 6), ("dec.o", *llm[1], 6), ("dec.gu", *llm[2], 6), ("dec.down", *llm[3], 6),
              ("dec.lm_head", cfg.vocab, cfg.width, 6), ("dn.gu", *exp[2], 50), ("dn.down", *exp[3], 50)]
    targets = [int(a) for a in sys.argv[1:]] or [68, 80]
    streams = [("all", torch.cuda.current_stream().cuda_stream, 148)]
    keep = []
    for n in targets:
        s, got, g = green_stream(n)
        keep.append(g)
        streams.append((f"{got} SMs", s, got))
    for name, n, k, t in shapes:
        sp = bench.policy_splits(1, n, k)
        copies = max(1, int(400e6 // (n * k * 2)))
        ws = [torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02 for _ in range(copies)]
        x = torch.randn(t, k, device="cuda", dtype=torch.bfloat16)
        o = torch.empty(t, n, device="cuda", dtype=torch.float32)
        wsp = torch.empty(max(1, sp * t * n), device="cuda", dtype=torch.float32)
        line = f"{name:12s} {n}x{k} T={t} splits={sp}:"
        for label, st, sms in streams:
            def call(w):
                _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
                          C.c_int32(k), C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n), None,
                          None, C.c_int32(0), C.c_int32(sp), C.c_void_p(wsp.data_ptr()), C.c_int64(wsp.numel()),
                          C.c_void_p(st))
            for w in ws[:2]:
                call(w)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ext = torch.cuda.ExternalStream(st)
            reps = 20
            e0.record(ext)
            for i in range(reps):
                call(ws[i % copies])
            e1.record(ext)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            line += f"  {label}: {us:7.1f} us {n * k * 2 / us / 1e3:6.0f} GB/s"
        print(line, flush=True)


if __name__ == "__main__":
    main()
