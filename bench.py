#!/usr/bin/env python
"""Headline benchmark: action Hz + concurrent language tokens/s per stream for a
pi0.5-shaped VLA (BASELINE.json configs[1]) through the unified-KV hot path.

One "step" = one control frame of ``run_frame_unified`` (Alg. 1): the frame's
new observation (3 x 224^2 cameras + 32 prompt tokens, P = 800) is prefilled
once into the paged KV pool, the action expert denoises a 50 x 32 chunk in 10
Euler steps off that shared prefix, and every live language request (budget
N = 30, k = 5 tokens per frame, steady batch B = N/k = 6) advances in one
continuously-batched decode.  ``--gpus N`` runs N independent stream groups
(one process per GPU, no collective on the hot path: weak scaling).

value : aggregate action Hz (H = 50) over all streams, inputs resident in HBM
e2e   : same metric through the public API with host (numpy) camera frames,
        H2D of frames + prompt ids and D2H of actions + tokens inside the
        timed region
--impl reference : the CPU restatement (oracle/pi05_ref.py, torch fp32) of
        the same frame on the host cores ("port"; the reference package has
        no pi0.5 model), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
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


def args_parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--streams", type=int, default=1, help="lock-stepped robot streams per GPU")
    p.add_argument("--total-streams", type=int, default=0,
                   help="shard this many streams over the ranks (stream s -> rank s mod N); "
                        "overrides --streams (BASELINE configs[4]: 64)")
    p.add_argument("--k", type=int, default=5, help="decode tokens per frame")
    p.add_argument("--budget", type=int, default=30, help="language tokens per request (N)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip e2e/roofline (profiler runs)")
    return p.parse_args()


# ----------------------------------------------------------------- plumbing

def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce(ws, value, op):
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
    return t.item()


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
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- workload

def frame_inputs(cfg, stream: int, frame: int, rng_seed: int = 1):
    """Deterministic synthetic observation for (stream, frame)."""
    from paper_2603_14371_b200.pi05 import synthetic_images
    from paper_2603_14371_b200.rng import SplitMix64
    seed = (rng_seed << 40) ^ (stream << 20) ^ frame
    r = SplitMix64(seed)
    toks = tuple(r.below(cfg.vocab) for _ in range(PROMPT))
    return toks, synthetic_images(N_CAMS, seed)


def build_frames(cfg, streams, n_frames, budget, device):
    """Arrivals per frame; images on device (value) or host (e2e)."""
    import torch
    from paper_2603_14371_b200.pi05 import Pi05Observation
    from paper_2603_14371_b200.workload import Arrival
    frames = []
    for f in range(n_frames):
        arr = []
        for s in range(streams):
            toks, imgs = frame_inputs(cfg, s, f)
            if device:
                imgs = torch.from_numpy(imgs).cuda()
            arr.append(Arrival(f, Pi05Observation(toks, f, imgs), budget))
        frames.append(arr)
    return frames


def run_frames(backend, frames, k, f_min=30.0):
    from paper_2603_14371_b200.kv_manager import KvManager
    from paper_2603_14371_b200.scheduler import run_frame_unified
    mgr = KvManager()
    traces = [run_frame_unified(t, arr, mgr, backend, k, f_min).trace for t, arr in enumerate(frames)]
    return traces, mgr


def timed(ws, backend, frames, warmup, k):
    """Run warmup frames, then time the rest with CUDA events (max over ranks)."""
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
        start.record()
        for t in range(warmup, len(frames)):
            traces.append(run_frame_unified(t, frames[t], mgr, backend, k, 30.0).trace)
        end.record()
        torch.cuda.synchronize()
    launches = _lib.lib().oxy_launch_count() - n0
    barrier(ws)
    ms = reduce(ws, start.elapsed_time(end), "max")
    return ms, traces, launches, clk.summary()


# ----------------------------------------------------------------- kernel rooflines

def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the roofline
    kernels, from one committed `ncu --set full` capture (tools/profile_all.sh)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def kernel_rooflines(backend, m_decode):
    """CUDA-event timings of single kernels at the frame's shapes."""
    import ctypes as C
    import torch
    from paper_2603_14371_b200 import _lib
    hbm, tf_burst, tf_sus, kind = peaks()
    cfg = backend.config
    st = torch.cuda.current_stream()
    out = {}
    tr = ncu_traffic()

    def traffic(key):
        return tr[key]["traffic_bytes"] if key in tr else None

    def time_launches(fn, n=20, warm=3):
        for _ in range(warm):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(n):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n / 1e3  # seconds per launch

    def gemm_fn(w, x, o, n, kk, t, splits=0):
        plan = (C.c_int32 * 6)()
        _lib.call("oxy_gemm_plan", C.c_int32(n), C.c_int32(kk), C.c_int32(t), C.c_int32(splits), plan)
        ws_t = torch.empty(max(1, plan[3] * t * n), dtype=torch.float32, device="cuda")
        args = (C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_int32(n), C.c_int32(kk),
                C.c_int32(t), C.c_int32(0), C.c_void_p(o.data_ptr()), C.c_int32(n), None, None,
                C.c_int32(0), C.c_int32(splits), C.c_void_p(ws_t.data_ptr()),
                C.c_int64(ws_t.numel()), C.c_void_p(st.cuda_stream))
        return lambda: _lib.call("oxy_gemm_bf16", *args), ws_t

    # 1. LM-head GEMM at the decode shape (largest single launch of a frame; HBM-bound)
    n, kk, t = cfg.vocab, cfg.width, max(1, m_decode)
    w = torch.randn(n, kk, device="cuda", dtype=torch.bfloat16)
    x = torch.randn(t, kk, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    fn, keep = gemm_fn(w, x, o, n, kk, t)
    sec = time_launches(fn)
    byts = n * kk * 2 + t * kk * 2 + t * n * 4
    out["gemm_lm_head"] = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": hbm, "unit": "GB/s",
                           "frac": byts / sec / 1e9 / hbm, "traffic": traffic("lm_head"),
                           "algorithmic_bytes": byts, "shape": f"{n}x{kk} bf16 weights, T={t}", "us": sec * 1e6,
                           "peak_kind": kind}
    del w, x, o, keep
    # 2. prefill FFN gate/up GEMM (tensor-bound): [2*mlp, width] x [800 tokens]
    n, kk, t = 2 * cfg.mlp, cfg.width, 800
    w = torch.randn(n, kk, device="cuda", dtype=torch.bfloat16) * 0.02
    x = torch.randn(t, kk, device="cuda", dtype=torch.bfloat16)
    o = torch.empty(t, n, device="cuda", dtype=torch.float32)
    fn, keep = gemm_fn(w, x, o, n, kk, t)
    sec = time_launches(fn)
    flops = 2.0 * n * kk * t
    out["gemm_prefill_ffn"] = {"bound": "tensor", "achieved": flops / sec / 1e12, "peak": tf_burst,
                               "unit": "TFLOP/s", "frac": flops / sec / 1e12 / tf_burst,
                               "traffic": traffic("prefill_gu"), "shape": f"{n}x{kk} x T={t}", "us": sec * 1e6,
                               "peak_kind": kind + " burst"}
    del w, x, o, keep
    # 3. paged decode attention: 64 rows x 1024-position contexts (MQA 8q/1kv, hd 256)
    rows, ctx, blk = 64, 1024, 64
    nb = rows * ctx // blk
    kp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    vp = torch.randn(nb, blk, 256, device="cuda", dtype=torch.bfloat16)
    perm = torch.randperm(nb, device="cuda", generator=None).to(torch.int32)
    bt = perm.reshape(rows, ctx // blk).contiguous()
    pos = torch.full((rows,), ctx - 1, dtype=torch.int32, device="cuda")
    q = torch.randn(rows, 2048, device="cuda", dtype=torch.bfloat16)
    ob = torch.empty_like(q)
    wsd = torch.empty(rows * (ctx // blk) * 8 * 258, device="cuda", dtype=torch.float32)
    args = (C.c_void_p(q.data_ptr()), C.c_void_p(ob.data_ptr()), C.c_void_p(kp.data_ptr()),
            C.c_void_p(vp.data_ptr()), C.c_int32(nb), C.c_void_p(bt.data_ptr()), C.c_int32(ctx // blk),
            C.c_void_p(pos.data_ptr()), C.c_int32(rows), C.c_int32(ctx // blk),
            C.c_void_p(wsd.data_ptr()), C.c_void_p(st.cuda_stream))
    sec = time_launches(lambda: _lib.call("oxy_paged_decode_attention", *args))
    byts = rows * ctx * 256 * 2 * 2 + rows * 2048 * 2 * 2
    out["decode_attention"] = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": hbm,
                               "unit": "GB/s", "frac": byts / sec / 1e9 / hbm, "traffic": traffic("decode_attn"),
                               "algorithmic_bytes": byts, "shape": f"{rows} rows x {ctx} ctx, 8q/1kv hd256 (incl. merge)",
                               "us": sec * 1e6, "peak_kind": kind}
    return out


# ----------------------------------------------------------------- CPU baseline

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


# ----------------------------------------------------------------- arms

def ours(a, ws, rank, local):
    import torch
    from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config
    cfg = Pi05Config()
    if a.total_streams:
        from paper_2603_14371_b200.sharding import streams_for_rank
        a.streams = max(1, len(streams_for_rank(a.total_streams, ws, rank)))
    r, k, budget = a.streams, a.k, a.budget
    steady_m = r * -(-budget // k)
    n_frames = a.warmup + a.steps
    backend = Pi05Backend(cfg, num_blocks=256 + r * 64, measure=True)
    frames_dev = build_frames(cfg, r, n_frames, budget, device=True)
    ms, traces, launches, clocks = timed(ws, backend, frames_dev, a.warmup, k)
    frames_total = a.steps * r
    tokens = sum(t.tokens_emitted for t in traces)
    tokens_all = reduce(ws, tokens, "sum")
    frames_all = reduce(ws, frames_total, "sum")
    sec = ms / 1e3
    value = H_REPORT * frames_all / sec
    streams_all = r * ws
    stage = {s: statistics.mean(getattr(t, s) for t in traces) / 1e3
             for s in ("prefill_us", "denoise_us", "decode_us")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: splitmix64 camera frames + prompt ids, random-init pi0.5-shaped "
                "weights (Gemma-2B + Gemma-300M expert + SigLIP So400m/14)",
        "config": {"workload": f"pi0.5 unified-KV frame loop, {r} stream(s)/GPU: {N_CAMS}x224^2 "
                               f"cams + {PROMPT} prompt tok (P=800), chunk H=50 A=32, S=10 Euler "
                               f"steps, lang budget N={budget} k={k}/frame (steady B={steady_m})",
                   "streams_per_gpu": r, "decode_k": k, "budget_N": budget,
                   "l2": "inputs larger than L2 (7.8 GB of weights streamed per frame)",
                   "parallelism": f"{ws} independent stream group(s), no collective"},
        "action_hz_per_stream": value / streams_all,
        "action_hz_per_stream_H10": value / streams_all * 10 / H_REPORT,
        "lang_tok_s_per_stream": tokens_all / sec / streams_all,
        "frame_ms": ms / a.steps,
        "stage_ms": {k_: round(v, 3) for k_, v in stage.items()},
        "steady_batch": statistics.mean(t.batch_size_m for t in traces),
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not a.no_extras:
        # the same frames with the stages run back to back (no denoise/decode overlap)
        backend.admit_overlapped = None
        s_ms, s_traces, _, _ = timed(ws, backend, frames_dev, a.warmup, k)
        del backend.admit_overlapped
        line["stage_serial"] = {
            "frame_ms": s_ms / a.steps, "value": H_REPORT * frames_all / (s_ms / 1e3),
            "stage_ms": {k_: round(statistics.mean(getattr(t, k_) for t in s_traces) / 1e3, 3)
                         for k_ in ("prefill_us", "denoise_us", "decode_us")}}
        frames_host = build_frames(cfg, r, n_frames, budget, device=False)
        backend.meter = None
        e_ms, e_traces, _, _ = timed(ws, backend, frames_host, a.warmup, k)
        e_sec = e_ms / 1e3
        img_bytes = N_CAMS * 224 * 224 * 3
        line["e2e"] = {
            "value": H_REPORT * reduce(ws, frames_total, "sum") / e_sec, "unit": UNIT,
            "h2d_bytes_per_step": r * (img_bytes + PROMPT * 4),
            "d2h_bytes_per_step": r * cfg.H * cfg.action_dim * 4 + 4 * k * steady_m,
            "lang_tok_s_per_stream": reduce(ws, sum(t.tokens_emitted for t in e_traces), "sum")
            / e_sec / streams_all,
            "path": "run_frame_unified(Pi05Backend) with numpy frames (public API)"}
        if rank == 0:
            rl = kernel_rooflines(backend, steady_m)
            line["roofline"] = rl["gemm_lm_head"]
            line["roofline"]["kernel"] = "gemm_sm100 (tcgen05) @ LM head"
            line["roofline_all"] = rl
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
    return line


def reference(a, ws, rank):
    if rank != 0:
        return None
    import torch
    from oracle.pi05_ref import Pi05Ref
    from paper_2603_14371_b200.pi05 import Pi05Config
    cfg = Pi05Config()
    cores = cpu_threads()
    k, budget = a.k, a.budget
    m = a.streams * -(-budget // k)
    ref = Pi05Ref.from_counter(cfg)
    for _ in range(a.warmup):
        cpu_frame(ref, cfg, k, m)
    t0 = time.perf_counter()
    toks = 0
    for _ in range(a.steps):
        _, n = cpu_frame(ref, cfg, k, m)
        toks += n
    sec = time.perf_counter() - t0
    value = H_REPORT * a.steps * a.streams / sec
    sample = (f"{a.steps} steady frames of oracle/pi05_ref.py (torch fp32, {cores} threads): "
              f"prefill P=800 + {cfg.S}-step denoise + {k} decode steps x {m} rows")
    return {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": ws,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": sec * 1e3 / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (same frames and weights as the GPU arm)",
            "config": {"workload": "pi0.5 unified-KV frame (CPU restatement)", "streams": a.streams},
            "lang_tok_s_per_stream": toks / sec / a.streams,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    a = args_parse()
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
