#!/usr/bin/env python
"""Headline benchmark: action Hz + concurrent language tokens/s per stream for a
pi0.5-shaped VLA (BASELINE.json configs[1]) through the unified-KV hot path.

One "step" = one control frame of ``run_frame_unified`` (Alg. 1): the frame's
new observation (3 x 224^2 cameras + 32 prompt tokens, P = 800) is prefilled
once into the paged KV pool, the action expert denoises a 50 x 32 chunk in 10
Euler steps off that shared prefix, and every live language request (budget
N = 30, k = 5 tokens per frame, steady batch B = N/k = 6) advances in one
continuously-batched decode.

--gpus N : N ranks, one process per GPU (launched by torchrun, or spawned by
        this script under torch.distributed.run when WORLD_SIZE is unset), each
        pinned to its share of the host cores.  Robot streams are independent:
        stream s runs on rank s mod N with no collective on the
        frame path; NCCL only for the barrier and the end-of-run reduction
        (paper_2603_14371_b200.sharding.reduce_metrics).  N = 1 runs configs[1]
        (1 stream); N > 1 defaults to configs[4] (--total-streams 64 sharded over
        the ranks: strong scaling).

value : aggregate action Hz (H = 50) over all streams, inputs resident in HBM
e2e   : the same metric through the public API with host (numpy) camera frames,
        H2D of frames + prompt ids and D2H of actions + tokens inside the
        timed region
roofline : the dominant kernel class of the frame — the skinny tcgen05 GEMMs
        of the decode and denoise chains, timed as the frame runs them: one
        decode step's and one denoise step's projections (distinct weights per
        layer, frame plans) replayed as a CUDA graph with PDL, CUDA events around
        each replay, L2 flushed before it, weighted k : S per frame (the
        each-launch-alone figure rides along as roofline.alone) — plus frame-level and denoise-chain entries against the ideal frame
         and per-kernel entries in roofline_all
cpu_baseline : oracle/pi05_ref.py (torch fp32, all host cores) on one frame
cpu_baseline_c1 : the REFERENCE's own ToyBackend (baseline/_ref, numpy) at
        configs[0] (C1) timed beside this package's CUDA toy on the same frame
--impl reference : the CPU restatement (oracle/pi05_ref.py) of the configs[1]
        frame on the host cores ("port": the reference has no pi0.5 model),
        rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "action Hz + concurrent lang tokens/s per stream (pi0.5-shape), 1/2/4/8 B200"
UNIT = "Hz"
H_REPORT = 50
PROMPT = 32
N_CAMS = 3
# BASELINE configs[0] / SURVEY.md §8d C1: the reference toy at d = 256, P = 800, k = 16
C1 = dict(L=2, d_model=256, n_heads=4, vocab=1024, eos_token=0, action_dim=32, H=50, S=10, seed=7)


def args_parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--streams", type=int, default=1, help="lock-stepped robot streams per GPU")
    p.add_argument("--total-streams", type=int, default=None,
                   help="shard this many streams over the ranks (stream s -> rank s mod N); "
                        "default 64 when N > 1 (BASELINE configs[4]), else --streams per GPU")
    p.add_argument("--k", type=int, default=5, help="decode tokens per frame")
    p.add_argument("--budget", type=int, default=30, help="language tokens per request (N)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip e2e/roofline (profiler runs)")
    a = p.parse_args(argv)
    if a.total_streams is None:
        a.total_streams = 64 if a.gpus > 1 else 0
    return a


# ----------------------------------------------------------------- plumbing

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_command(argv, gpus: int, port: int) -> list[str]:
    """The driver's own launch line: one rank per GPU under torch.distributed.run."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def host_cores_for(local: int, nlocal: int, cores: list[int]) -> list[int]:
    """Disjoint, equal shares of the host cores per local rank (the Python frame
    orchestration of one rank must not contend with another's)."""
    cores = sorted(cores)
    per = max(1, len(cores) // max(1, nlocal))
    mine = cores[local * per:(local + 1) * per]
    return mine or cores


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if ws > 1:
        import torch.distributed as dist
        nlocal = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
        try:
            mine = host_cores_for(local, nlocal, list(os.sched_getaffinity(0)))
            os.sched_setaffinity(0, mine)
            torch.set_num_threads(len(mine))
        except (AttributeError, OSError):
            pass
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def aggregate(ws, elapsed_ms, stream_frames, tokens, streams, device="cuda"):
    """Whole-job numbers: time = max over ranks, counts summed (sharding.reduce_metrics;
    NCCL on the GPU box, gloo in tests/test_multiproc.py)."""
    from paper_2603_14371_b200.sharding import reduce_metrics
    return reduce_metrics(elapsed_ms / 1e3, stream_frames, tokens, streams, H_REPORT,
                          device=device if ws > 1 else "cpu")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    """(HBM GB/s, bf16 TF/s burst, bf16 TF/s sustained, source)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained") or p["bf16_tflops"], "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- workload

def frame_inputs(cfg, stream: int, frame: int, rng_seed: int = 1):
    """Deterministic synthetic observation for (stream, frame)."""
    from paper_2603_14371_b200.pi05 import synthetic_images
    from paper_2603_14371_b200.rng import SplitMix64
    seed = (rng_seed << 40) ^ (stream << 20) ^ frame
    r = SplitMix64(seed)
    toks = tuple(r.below(cfg.vocab) for _ in range(PROMPT))
    return toks, synthetic_images(N_CAMS, seed)


def build_frames(cfg, streams, n_frames, budget, device, stream0=0):
    """Arrivals per frame (one per stream of this rank); images on device (value)
    or host (e2e)."""
    import torch
    from paper_2603_14371_b200.pi05 import Pi05Observation
    from paper_2603_14371_b200.workload import Arrival
    frames = []
    for f in range(n_frames):
        arr = []
        for s in streams:
            toks, imgs = frame_inputs(cfg, s, f)
            if device:
                imgs = torch.from_numpy(imgs).cuda()
            arr.append(Arrival(f, Pi05Observation(toks, f, imgs), budget))
        frames.append(arr)
    return frames


def timed(ws, backend, frames, warmup, k):
    """Run warmup frames, then time the rest with CUDA events on the backend's
    stream (the caller-side current stream every stage joins back into)."""
    import torch
    from paper_2603_14371_b200 import _lib
    from paper_2603_14371_b200.kv_manager import KvManager
    from paper_2603_14371_b200.scheduler import run_frame_unified
    mgr = KvManager()
    for t in range(warmup):
        run_frame_unified(t, frames[t], mgr, backend, k, 30.0)
    torch.cuda.synchronize()
    barrier(ws)
    n0 = _lib.lib().oxy_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    traces = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        start.record()
        for t in range(warmup, len(frames)):
            traces.append(run_frame_unified(t, frames[t], mgr, backend, k, 30.0).trace)
        end.record()
        torch.cuda.synchronize()
    launches = _lib.lib().oxy_launch_count() - n0
    barrier(ws)
    return start.elapsed_time(end), traces, launches, clk.summary()


# ----------------------------------------------------------------- ideal frame

def projections(cfg):
    """(n_out, K) of every projection per layer, per tower."""
    qkv, qdim = 10 * 256, 8 * 256
    llm = [(qkv, cfg.width), (cfg.width, qdim), (2 * cfg.mlp, cfg.width), (cfg.width, cfg.mlp)]
    exp = [(qkv, cfg.expert_width), (cfg.expert_width, qdim), (2 * cfg.expert_mlp, cfg.expert_width),
           (cfg.expert_width, cfg.expert_mlp)]
    vit = [(3 * cfg.vit_width, cfg.vit_width), (cfg.vit_width, cfg.vit_width), (cfg.vit_mlp, cfg.vit_width),
           (cfg.vit_width, cfg.vit_mlp)]
    return llm, exp, vit


def ideal_frame(cfg, r, k, m, P, ctx):
    """Serial ideal time of one frame on one GPU: prefill at the sustained tensor
    peak, denoise and decode at the HBM peak (weights once per Euler / decode step,
    plus the prefix / context KV each step reads: 18 432 B per position)."""
    hbm, _, tf_sus, _ = peaks()
    llm, exp, vit = projections(cfg)
    n_llm = cfg.depth * sum(a * b for a, b in llm)
    n_exp = cfg.depth * sum(a * b for a, b in exp)
    n_vit = cfg.vit_depth * sum(a * b for a, b in vit) + cfg.vit_width * 588 + cfg.width * cfg.vit_width
    kv_pos = 2 * cfg.depth * 256 * 2
    t_img = 256 * N_CAMS
    pf_flops = r * (2 * n_llm * P + cfg.depth * 8 * 4 * P * P * 256
                    + 2 * n_vit * t_img + cfg.vit_depth * cfg.vit_heads * 4 * 256 * 256 * 72 * N_CAMS)
    dn_bytes = cfg.S * (2 * n_exp + r * kv_pos * (P + cfg.H))
    dec_bytes = k * (2 * (n_llm + cfg.vocab * cfg.width) + m * kv_pos * ctx)
    out = {"prefill_ms": pf_flops / (tf_sus * 1e12) * 1e3, "denoise_ms": dn_bytes / (hbm * 1e9) * 1e3,
           "decode_ms": dec_bytes / (hbm * 1e9) * 1e3, "prefill_tflop": pf_flops / 1e12,
           "denoise_gb": dn_bytes / 1e9, "decode_gb": dec_bytes / 1e9}
    out["total_ms"] = out["prefill_ms"] + out["denoise_ms"] + out["decode_ms"]
    return out


# ----------------------------------------------------------------- kernel rooflines

def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the roofline
    kernels, from one committed `ncu --set full` capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


class ColdTimer:
    """Per-launch CUDA-event timing with an L2 flush (a 512 MB write, 4x the L2)
    before every launch, so weights and KV stream from HBM as in the frame."""

    def __init__(self):
        import torch
        self.torch = torch
        self.flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def __call__(self, fn, n=10, warm=2):
        torch = self.torch
        for _ in range(warm):
            fn()
        pairs = []
        for _ in range(n):
            self.flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            pairs.append((s, e))
        torch.cuda.synchronize()
        return statistics.mean(s.elapsed_time(e) for s, e in pairs) / 1e3  # seconds per launch


def gemm_launcher(n, kk, t, mode, splits):
    """oxy_gemm_bf16 at a given plan: returns (fn, keep-alive tensors)."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    st = torch.cuda.current_stream()
    w = torch.randn(n, kk, device="cuda", dtype=torch.bfloat16) * 0.02
    x = torch.randn(t, kk, device="cuda", dtype=torch.bfloat16)
    o = torch.zeros(t, n if mode != 3 else n // 2, device="cuda",
                    dtype=torch.float32 if mode in (0, 2) else torch.bfloat16)
    ws_t = torch.empty(max(1, splits * t * n), dtype=torch.float32, device="cuda")
    args = (C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(kk), C.c_int32(t),
            C.c_int32(mode), C.c_void_p(o.data_ptr()), C.c_int32(o.shape[1]), None, None, C.c_int32(0),
            C.c_int32(splits), C.c_void_p(ws_t.data_ptr()), C.c_int64(ws_t.numel()), C.c_void_p(st.cuda_stream))
    return (lambda: _lib.call("oxy_gemm_bf16", *args)), (w, x, o, ws_t)


def policy_splits(phase, n, kk):
    import ctypes as C
    from paper_2603_14371_b200 import _lib
    s = C.c_int32()
    _lib.call("oxy_gemm_policy_splits", C.c_int32(phase), C.c_int32(n), C.c_int32(kk), C.byref(s))
    return s.value


def skinny_gemm_class(cfg, m_decode, r, k, timer, hbm, kind):
    """The frame's dominant kernel class: the skinny tcgen05 GEMMs of the decode
    chain (T = batch rows) and the denoise chain (T = 50 x streams), each at the
    frame's own plan (batch-invariant split-K, split reduce included), timed
    alone after an L2 flush; the class entry weights each shape by its launches
    per frame (decode: k steps x depth, LM head k; denoise: S steps x depth)."""
    llm, exp, _ = projections(cfg)
    names = ("qkv", "o", "gate_up", "down")
    modes = (1, 2, 3, 2)  # bf16 out, f32 +=, GeGLU, f32 += (the frame fuses RoPE / residual + norm)
    shapes = [(f"decode.{nm}", n, kk, m_decode, md, k * cfg.depth) for nm, (n, kk), md in zip(names, llm, modes)]
    shapes.append(("decode.lm_head", cfg.vocab, cfg.width, m_decode, 0, k))
    shapes += [(f"denoise.{nm}", n, kk, cfg.H * r, md, cfg.S * cfg.depth)
               for nm, (n, kk), md in zip(names, exp, modes)]
    entries, tot_b, tot_s = {}, 0.0, 0.0
    traffic = ncu_traffic().get("skinny_shapes", {})
    for name, n, kk, t, mode, per_frame in shapes:
        sp = policy_splits(1, n, kk)
        fn, keep = gemm_launcher(n, kk, t, mode, sp)
        sec = timer(fn)
        byts = n * kk * 2 + t * kk * 2 + t * (n // 2 if mode == 3 else n) * (4 if mode in (0, 2) else 2)
        entries[name] = {"achieved": byts / sec / 1e9, "frac": byts / sec / 1e9 / hbm, "us": sec * 1e6,
                         "algorithmic_bytes": byts, "shape": f"{n}x{kk} T={t} splits={sp}",
                         "launches_per_frame": per_frame,
                         "traffic": traffic.get(name, {}).get("traffic_bytes")}
        tot_b += byts * per_frame
        tot_s += sec * per_frame
        del keep
    ach = tot_b / tot_s / 1e9
    cls = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
           "traffic": ncu_traffic().get("skinny_class", {}).get("traffic_bytes_per_frame"),
           "kernel": "gemm_sm100 gemm_kernel (tcgen05, split-K + reduce) — decode and denoise chains",
           "algorithmic_bytes": tot_b, "unit_of_work": "one frame's skinny GEMM launches",
           "launch_ms_per_frame": tot_s * 1e3, "peak_kind": kind,
           "timing": "each launch alone, CUDA events, L2 flushed (512 MB write) before every launch"}
    return cls, entries


def skinny_gemm_chain(cfg, m_decode, r, k, hbm, kind):
    """The same skinny GEMM class in its chain: one decode step's projections
    (depth x {qkv, o, gate/up, down} at T = batch rows, then the LM head) and one
    denoise step's (depth x 4 at T = 50 x streams), each layer with its own weights
    (4.9 GB / 0.6 GB per chain, far above L2), captured into a CUDA graph and replayed
    back to back on one stream with PDL, as the frame issues them — minus the
    attention and norm kernels between them.  Time per chain by CUDA events around
    the replay (L2 flushed before each); the class figure weights the two chains by
    the frame's k decode and S denoise steps."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    llm, exp, _ = projections(cfg)
    modes = (1, 2, 3, 2)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for name, shapes, t, per_frame in (
            ("decode_step", [(n, kk, md) for _ in range(cfg.depth) for (n, kk), md in zip(llm, modes)]
             + [(cfg.vocab, cfg.width, 0)], m_decode, k),
            ("denoise_step", [(n, kk, md) for _ in range(cfg.depth) for (n, kk), md in zip(exp, modes)],
             cfg.H * r, cfg.S)):
        keep, byts = [], 0
        x = torch.randn(t, max(kk for _, kk, _ in shapes), device="cuda", dtype=torch.bfloat16)
        plans = []
        for n, kk, md in shapes:
            w = torch.empty(n, kk, device="cuda", dtype=torch.bfloat16).normal_(0, 0.02)
            o = torch.zeros(t, n if md != 3 else n // 2, device="cuda",
                            dtype=torch.float32 if md in (0, 2) else torch.bfloat16)
            sp = policy_splits(1, n, kk)
            ws_t = torch.empty(max(1, sp * t * n), dtype=torch.float32, device="cuda")
            keep += [w, o, ws_t]
            plans.append((w, o, ws_t, n, kk, md, sp))
            byts += n * kk * 2 + t * kk * 2 + t * (n // 2 if md == 3 else n) * (4 if md in (0, 2) else 2)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            for _ in range(2):  # eager warm-up (plans, tensor maps) before capture
                for w, o, ws_t, n, kk, md, sp in plans:
                    _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
                              C.c_int32(kk), C.c_int32(t), C.c_int32(md), C.c_void_p(o.data_ptr()),
                              C.c_int32(o.shape[1]), None, None, C.c_int32(0), C.c_int32(sp),
                              C.c_void_p(ws_t.data_ptr()), C.c_int64(ws_t.numel()), C.c_void_p(side.cuda_stream))
        side.synchronize()
        with torch.cuda.graph(g, stream=side):
            cs = torch.cuda.current_stream().cuda_stream
            for w, o, ws_t, n, kk, md, sp in plans:
                _lib.call("oxy_gemm_bf16", C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n),
                          C.c_int32(kk), C.c_int32(t), C.c_int32(md), C.c_void_p(o.data_ptr()),
                          C.c_int32(o.shape[1]), None, None, C.c_int32(0), C.c_int32(sp),
                          C.c_void_p(ws_t.data_ptr()), C.c_int64(ws_t.numel()), C.c_void_p(cs))
        for _ in range(3):
            g.replay()
        pairs = []
        for _ in range(10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            pairs.append((s, e))
        torch.cuda.synchronize()
        sec = statistics.mean(s.elapsed_time(e) for s, e in pairs) / 1e3
        out[name] = {"achieved": byts / sec / 1e9, "frac": byts / sec / 1e9 / hbm, "ms": sec * 1e3,
                     "launches": len(shapes), "T": t, "algorithmic_bytes": byts, "per_frame": per_frame}
        del g, keep, plans, x
        torch.cuda.empty_cache()
    tot_b = sum(v["algorithmic_bytes"] * v["per_frame"] for v in out.values())
    tot_s = sum(v["ms"] / 1e3 * v["per_frame"] for v in out.values())
    ach = tot_b / tot_s / 1e9
    cls = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
           "kernel": "gemm_sm100 gemm_kernel (tcgen05, split-K + reduce) — decode and denoise chains",
           "algorithmic_bytes": tot_b, "unit_of_work": "one frame's skinny GEMM launches",
           "launch_ms_per_frame": tot_s * 1e3, "peak_kind": kind,
           "timing": "in chain: each step's projections replayed as one CUDA graph with PDL, "
                     "distinct weights per layer, L2 flushed before each replay", "chains": out}
    return cls


def kernel_rooflines(cfg, m_decode, r, k):
    """Per-kernel rooflines (CUDA events inside bench.py) at the frame's shapes."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    hbm, tf_burst, _, kind = peaks()
    timer = ColdTimer()
    tr = ncu_traffic()
    out = {}
    cls, entries = skinny_gemm_class(cfg, m_decode, r, k, timer, hbm, kind)
    out["skinny_gemm_class"] = cls
    out["skinny_gemm_shapes"] = entries
    out["skinny_gemm_chain"] = skinny_gemm_chain(cfg, m_decode, r, k, hbm, kind)
    # prefill FFN gate/up GEMM (tensor-bound): [2*mlp, width] x [800 tokens], persistent 2-CTA kernel
    n, kk, t = 2 * cfg.mlp, cfg.width, 800
    fn, keep = gemm_launcher(n, kk, t, 3, policy_splits(0, n, kk))
    sec = timer(fn)
    flops = 2.0 * n * kk * t
    out["gemm_prefill_gate_up"] = {"bound": "tensor", "achieved": flops / sec / 1e12, "peak": tf_burst,
                                   "unit": "TFLOP/s", "frac": flops / sec / 1e12 / tf_burst,
                                   "traffic": tr.get("prefill_gu", {}).get("traffic_bytes"),
                                   "shape": f"{n}x{kk} x T={t}", "us": sec * 1e6, "peak_kind": kind + " burst"}
    del keep
    # paged decode attention at >= 256 MB per launch: 256 rows x 1024-position contexts
    st = torch.cuda.current_stream()
    rows, ctx, blk = 256, 1024, 64
    nb = rows * ctx // blk
    kp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    bt = torch.randperm(nb, device="cuda").to(torch.int32).reshape(rows, ctx // blk).contiguous()
    pos = torch.full((rows,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, 2048, device="cuda", dtype=torch.bfloat16)
    ob = torch.empty_like(q)
    wsd = torch.empty(rows * (ctx // blk) * 8 * 258, device="cuda", dtype=torch.float32)
    args = (C.c_void_p(q.data_ptr()), C.c_void_p(ob.data_ptr()), C.c_void_p(kp.data_ptr()),
            C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()), C.c_int32(ctx // blk),
            C.c_void_p(pos.data_ptr()), C.c_int32(rows), C.c_int32(ctx // blk),
            C.c_void_p(wsd.data_ptr()), C.c_void_p(st.cuda_stream))
    sec = timer(lambda: _lib.call("oxy_paged_decode_attention", *args))
    byts = rows * ctx * 256 * 2 * 2 + rows * 2048 * 2 * 2
    out["decode_attention"] = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": byts / sec / 1e9 / hbm,
                               "traffic": tr.get("decode_attn", {}).get("traffic_bytes"),
                               "algorithmic_bytes": byts,
                               "shape": f"{rows} rows x {ctx} ctx, 8q/1kv hd256 (incl. merge), L2 flushed",
                               "us": sec * 1e6, "peak_kind": kind}
    return out


# ----------------------------------------------------------------- CPU baselines

def cpu_frame(ref, cfg, k, m_decode):
    """One steady-state frame of the oracle on the host: prefill + S-step
    denoise + k decode steps for m_decode rows.  Returns (seconds, tokens)."""
    from paper_2603_14371_b200.pi05 import Pi05Observation
    toks, imgs = frame_inputs(cfg, 0, 0)
    obs = Pi05Observation(toks, 0, imgs)
    t0 = time.perf_counter()
    kvs = ref.prefill(obs)
    ref.denoise(kvs, cfg.S)
    ref.decode_rows([kvs] * m_decode, [cfg.eos_token] * m_decode, k)
    return time.perf_counter() - t0, m_decode * k


def cpu_threads():
    import torch
    n = len(os.sched_getaffinity(0))
    torch.set_num_threads(n)
    return n


def c1_frame_legs(frames=3):
    """configs[0] (C1): one Unified frame — prefill of the 800-token observation,
    10-step denoise, 16-token decode — of the REFERENCE ToyBackend (numpy, from
    baseline/_ref) on the host, and of this package's CUDA toy on the GPU, same
    arrival, same weights (the splitmix64 draw order), same greedy tokens."""
    import importlib
    import torch
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "kvweaver")):
        return {"unavailable": "reference not installed (sh tools/install_reference.sh)"}
    sys.path.insert(0, ref_dir)
    try:
        kw = importlib.import_module("kvweaver")
        ksched = importlib.import_module("kvweaver.scheduler")
    finally:
        sys.path.remove(ref_dir)
    from paper_2603_14371_b200 import BackendConfig, KvManager, WorkloadSpec, generate_arrivals
    from paper_2603_14371_b200.scheduler import run_frame_unified
    from paper_2603_14371_b200.toy_b200 import ToyBackend
    spec = dict(pattern="OnePerFrame", default_N=16, obs_len=800, num_frames=1, seed=1)
    ref_be = kw.ToyBackend(kw.BackendConfig(**C1))
    ref_arr = kw.generate_arrivals(kw.WorkloadSpec(**spec), C1["vocab"])[0]
    ref_ms, ref_tok = [], None
    for _ in range(frames):
        t0 = time.perf_counter()
        res = ksched.run_frame_unified(0, [ref_arr], kw.KvManager(), ref_be, 16, 30.0)
        ref_ms.append((time.perf_counter() - t0) * 1e3)
        ref_tok = res.finished[0][1] if res.finished else None
    gpu_be = ToyBackend(BackendConfig(**C1))
    arr = generate_arrivals(WorkloadSpec(**spec), C1["vocab"])[0]
    gpu_ms, gpu_tok = [], None
    for i in range(frames + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_frame_unified(0, [arr], KvManager(), gpu_be, 16, 30.0)
        torch.cuda.synchronize()
        if i >= 2:
            gpu_ms.append((time.perf_counter() - t0) * 1e3)
        gpu_tok = res.finished[0][1] if res.finished else None
    r, g = statistics.median(ref_ms), statistics.median(gpu_ms)
    return {"config": "configs[0] / C1: ToyBackend(L=2, d=256, 4 heads, V=1024, H=50, S=10, seed=7), "
                      "one Unified frame: prefill P=800 + 10-step denoise + 16-token decode",
            "reference_cpu_ms": r, "cores": len(os.sched_getaffinity(0)), "kind": "reference",
            "impl": "kvweaver.ToyBackend (numpy float64, unmodified, baseline/_ref)",
            "gpu_f1_ms": g, "gpu_impl": "ToyBackend over liboxygen_b200.so (fp32 verification mode)",
            "speedup": r / g, "tokens_equal": ref_tok == gpu_tok and ref_tok is not None,
            "sample": f"median of {frames} frames each (wall clock around run_frame_unified)"}


# ----------------------------------------------------------------- arms

def ours(a, ws, rank, local):
    import torch
    from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config
    from paper_2603_14371_b200.sharding import streams_for_rank
    cfg = Pi05Config()
    if a.total_streams:
        mine = streams_for_rank(a.total_streams, ws, rank)
        scaling = "strong"
    else:
        mine = list(range(rank * a.streams, (rank + 1) * a.streams))
        scaling = "weak"
    r, k, budget = len(mine), a.k, a.budget
    steady_m = r * -(-budget // k)
    n_frames = a.warmup + a.steps
    backend = Pi05Backend(cfg, num_blocks=256 + r * 96, measure=True)
    frames_dev = build_frames(cfg, mine, n_frames, budget, device=True)
    # the headline run without the stage meter (its CUDA-event reads synchronise the
    # host every frame); stage times from a second, instrumented run of the same frames
    meter, backend.meter = backend.meter, None
    ms, traces, launches, clocks = timed(ws, backend, frames_dev, a.warmup, k)
    backend.meter = meter
    tokens = sum(t.tokens_emitted for t in traces)
    agg = aggregate(ws, ms, a.steps * r, tokens, r)
    value = agg["action_hz"]
    streams_all = agg["streams"]
    m_ms, m_traces, _, _ = timed(ws, backend, frames_dev, a.warmup, k)
    stage = {s: statistics.mean(getattr(t, s + "_us") for t in m_traces) / 1e3
             for s in ("prefill", "denoise", "decode")}
    ideal = ideal_frame(cfg, r, k, steady_m, 800, 800 + budget // 2)
    dec_w_gb = k * (2 * sum(a_ * b_ for a_, b_ in projections(cfg)[0]) * cfg.depth + 2 * cfg.vocab * cfg.width) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": agg["elapsed_s"] * 1e3 / a.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: splitmix64 camera frames + prompt ids, random-init pi0.5-shaped "
                "weights (Gemma-2B + Gemma-300M expert + SigLIP So400m/14)",
        "config": {"workload": f"pi0.5 unified-KV frame loop, {r} stream(s) on this GPU"
                               f"{f' of {a.total_streams} sharded over {ws}' if a.total_streams else ''}: "
                               f"{N_CAMS}x224^2 cams + {PROMPT} prompt tok (P=800), chunk H=50 A=32, S=10 "
                               f"Euler steps, lang budget N={budget} k={k}/frame (steady B={steady_m})",
                   "streams_per_gpu": r, "total_streams": streams_all, "decode_k": k, "budget_N": budget,
                   "l2": f"inputs larger than L2: ~{dec_w_gb + ideal['denoise_gb']:.0f} GB of weights "
                         f"streamed per frame (decode {k} x 5.0 GB, denoise {cfg.S} x 0.62 GB) vs 126 MB L2",
                   "parallelism": f"{ws} independent stream group(s), one process per GPU, no collective "
                                  f"on the frame path"},
        "action_hz_per_stream": agg["action_hz_per_stream"],
        "action_hz_per_stream_H10": agg["action_hz_per_stream"] * 10 / H_REPORT,
        "lang_tok_s_per_stream": agg["tok_s_per_stream"],
        "frame_ms": ms / a.steps,
        "stage_ms": {k_: round(v, 3) for k_, v in stage.items()},
        "stage_ms_note": f"instrumented run of the same frames ({m_ms / a.steps:.3f} ms/frame with the "
                         f"per-frame stage-event reads); denoise counted from the prefill's start "
                         f"(its first Euler step runs under the prefill, layer by layer)",
        "steady_batch": statistics.mean(t.batch_size_m for t in traces),
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not a.no_extras:
        frames_host = build_frames(cfg, mine, n_frames, budget, device=False)
        meter, backend.meter = backend.meter, None
        e_ms, e_traces, _, _ = timed(ws, backend, frames_host, a.warmup, k)
        backend.meter = meter
        e_agg = aggregate(ws, e_ms, a.steps * r, sum(t.tokens_emitted for t in e_traces), r)
        img_bytes = N_CAMS * 224 * 224 * 3
        line["e2e"] = {
            "value": e_agg["action_hz"], "unit": UNIT,
            "h2d_bytes_per_step": r * (img_bytes + PROMPT * 4),
            "d2h_bytes_per_step": r * cfg.H * cfg.action_dim * 4 + 4 * k * steady_m,
            "lang_tok_s_per_stream": e_agg["tok_s_per_stream"],
            "path": "run_frame_unified(Pi05Backend) with numpy frames (public API)"}
        # the same frames with the stages run back to back (no denoise/decode overlap)
        backend.admit_overlapped = None
        s_ms, s_traces, _, _ = timed(ws, backend, frames_dev, a.warmup, k)
        del backend.admit_overlapped
        s_stage = {k_: statistics.mean(getattr(t, k_ + "_us") for t in s_traces) / 1e3
                   for k_ in ("prefill", "denoise", "decode")}
        line["stage_serial"] = {"frame_ms": s_ms / a.steps,
                                "value": aggregate(ws, s_ms, a.steps * r, 0, r)["action_hz"],
                                "stage_ms": {k_: round(v, 3) for k_, v in s_stage.items()}}
        backend.meter = None
        if rank == 0:
            hbm, _, tf_sus, kind = peaks()
            rl = kernel_rooflines(cfg, steady_m, r, k)
            # headline: the skinny GEMM class as the frame runs it (its chains, CUDA graph +
            # PDL); the per-launch-alone figure stays beside it in roofline_all
            line["roofline"] = dict(rl["skinny_gemm_chain"], alone={
                k_: rl["skinny_gemm_class"][k_] for k_ in ("achieved", "frac", "launch_ms_per_frame", "timing")})
            frame_ms = ms / a.steps
            line["roofline_all"] = dict(rl, frame={
                "bound": "mixed", "ideal_ms": ideal["total_ms"], "measured_ms": frame_ms,
                "frac": ideal["total_ms"] / frame_ms, "ideal": ideal,
                "note": "serial ideal: prefill at the sustained tensor peak, denoise and decode at HBM peak"},
                denoise_chain={
                "bound": "hbm", "achieved": ideal["denoise_gb"] / (s_stage["denoise"] / 1e3), "peak": hbm,
                "unit": "GB/s", "frac": ideal["denoise_ms"] / s_stage["denoise"],
                "ideal_ms": ideal["denoise_ms"], "measured_ms": s_stage["denoise"],
                "algorithmic_bytes": ideal["denoise_gb"] * 1e9,
                "note": f"{cfg.S} Euler steps x {r} stream(s), stage-serial frame (denoise alone)"})
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        from oracle.pi05_ref import Pi05Ref
        cores = cpu_threads()
        ref = Pi05Ref.from_backend(backend)
        del backend
        torch.cuda.empty_cache()
        sec_cpu, toks = cpu_frame(ref, cfg, k, steady_m)
        line["cpu_baseline"] = {
            "value": H_REPORT / sec_cpu, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"1 steady frame of oracle/pi05_ref.py (torch fp32): prefill P=800 + "
                      f"{cfg.S}-step denoise + {k} decode steps x {steady_m} rows "
                      f"({sec_cpu:.1f} s, {toks / sec_cpu:.2f} tok/s)"}
        del ref
        line["cpu_baseline_c1"] = c1_frame_legs()
    return line


def reference(a, ws, rank):
    if rank != 0:
        return None
    from oracle.pi05_ref import Pi05Ref
    from paper_2603_14371_b200.pi05 import Pi05Config
    cfg = Pi05Config()
    cores = cpu_threads()
    k, budget = a.k, a.budget
    streams = a.streams if not a.total_streams else max(1, a.total_streams // max(1, ws))
    m = streams * -(-budget // k)
    ref = Pi05Ref.from_counter(cfg)
    for _ in range(a.warmup):
        cpu_frame(ref, cfg, k, m)
    t0 = time.perf_counter()
    toks = 0
    for _ in range(a.steps):
        _, n = cpu_frame(ref, cfg, k, m)
        toks += n
    sec = time.perf_counter() - t0
    value = H_REPORT * a.steps / sec
    sample = (f"{a.steps} steady frames of oracle/pi05_ref.py (torch fp32, {cores} threads): "
              f"prefill P=800 + {cfg.S}-step denoise + {k} decode steps x {m} rows (1 stream's prefill "
              f"and denoise per frame)")
    return {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": ws,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": sec * 1e3 / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (same frames and weights as the GPU arm)",
            "config": {"workload": "pi0.5 unified-KV frame (CPU restatement of configs[1])", "streams": 1},
            "lang_tok_s_per_stream": toks / sec,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    a = args_parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without torchrun: launch N ranks exactly as the driver does
        sys.exit(subprocess.call(spawn_command(sys.argv[1:], a.gpus, free_port())))
    if a.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if a.steps > 3:  # each CPU frame takes seconds: keep the run within minutes
            a.steps, a.warmup = 3, min(a.warmup, 1)
        line = reference(a, ws, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    ws, rank, local = dist_init()
    line = ours(a, ws, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
