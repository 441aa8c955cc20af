"""Persistent wide GEMM: one CTA pair per unit (CL = 1) vs clusters of two pairs
multicasting the weight tile (CL = 2), at the prefill shapes.  Each variant runs in
its own process (the knobs are read once); prints us, TF/s and an output digest
(the two must be bit-identical: same K order).
    python tools/wide_cl_probe.py [K=V,K=V ...]   # parent: default / CL=2, or the given env variants
    (PROBE_SHAPES=gu800,qkv6400 restricts the shapes)
    python tools/wide_cl_probe.py child      # one variant (env knobs)"""
import ctypes as C
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = [("gu", 32768, 2048, 800, 3), ("gu", 32768, 2048, 1600, 3), ("gu", 32768, 2048, 6400, 3),
          ("down", 2048, 16384, 6400, 0), ("qkv", 2560, 2048, 6400, 1), ("vit.fc1", 4304, 1152, 6144, 1)]


def child():
    import torch
    from paper_2603_14371_b200 import _lib
    st = torch.cuda.current_stream()
    g = torch.Generator(device="cpu").manual_seed(5)
    only = [x for x in os.environ.get("PROBE_SHAPES", "").split(",") if x]
    for name, n, k, t, mode in SHAPES:
        if only and f"{name}{t}" not in only:
            continue
        w = (torch.randn(n, k, generator=g) * 0.02).to(torch.bfloat16).cuda()
        x = torch.randn(t, k, generator=g).to(torch.bfloat16).cuda()
        cols = n // 2 if mode == 3 else n
        o = torch.zeros(t, cols, device="cuda", dtype=torch.float32 if mode == 0 else torch.bfloat16)
        plan = (C.c_int32 * 6)()
        _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(k), C.c_int32(t), C.c_int32(0), plan)
        ws = torch.empty(max(1, plan[3] * t * n), device="cuda", dtype=torch.float32)
        f = lambda: _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
                              C.c_int32(k), C.c_int32(t), C.c_int32(mode), C.c_void_p(o.data_ptr()), C.c_int32(cols),
                              None, None, C.c_int32(0), C.c_int32(0), C.c_void_p(ws.data_ptr()),
                              C.c_int64(ws.numel()), C.c_void_p(st.cuda_stream))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        digest = hashlib.sha1(o.view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:12]
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / 10 * 1e3
        print(f"{name:8s} {n}x{k} T={t:5d} {us:8.1f} us {2 * n * k * t / us / 1e6:7.1f} TF/s plan={list(plan)} "
              f"digest={digest}", flush=True)


def main(variants):
    envs = [dict(kv.split("=") for kv in v.split(",") if kv) for v in variants] or [{}, {"OXY_GEMM_WIDE_CL": "2"}]
    for env in envs:
        print("#", env or "default", flush=True)
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "child"], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=300)
        print(r.stdout + r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    child() if sys.argv[1:] == ["child"] else main(sys.argv[1:])
