"""Cost-model calibration from measured B200 stage times.

The reference prices every stage with integer-microsecond constants
(``CostModelParams``, ``kvweaver/backend.py:125-160``):

    prefill(P)      = c_prefill_per_token * P
    denoise(S)      = S * c_denoise_per_step
    decode(k, m)    = k * (c_decode_base + c_decode_per_request * m)
    IsolatedParallel frame = max(p + a, p + d) * c_contention

``fit_cost_params`` fits those constants to CUDA-event stage timings (least
squares; the prefill and denoise lines through the origin as the model has no
intercept there); ``measure_stage_samples`` takes the timings on the GPU backend
at a spread of shapes.  With the fitted constants the reference's own
cost-model machinery (``run_simulation`` with ``backend_kind="CostModel"``,
``kvweaver/sim_engine.py:99``) reproduces the sweeps of
``tests/test_acceptance.py:145-200`` with B200 numbers instead of the paper's
RTX 4090 calibration, and ``closed_form_speedup`` predicts the Unified vs
IsolatedSequential frame-time ratio that tools/config_sweep.py measures.
"""

from __future__ import annotations

from .backend import CostModelParams

__all__ = ["fit_cost_params", "measure_stage_samples", "closed_form_speedup"]


def _through_origin(xy):
    sxx = sum(x * x for x, _ in xy)
    if sxx <= 0:
        raise ValueError("need at least one sample with a nonzero size")
    return sum(x * y for x, y in xy) / sxx


def fit_cost_params(prefill, denoise, decode, contention: float = 1.0) -> CostModelParams:
    """prefill: [(P, us)], denoise: [(S, us)], decode: [(k, m, us)] -> CostModelParams.

    Decode is fitted per step: us / k = base + per_request * m (ordinary least
    squares over m; needs >= 2 distinct m).  Constants are rounded to integer us
    and clamped at 0 as the reference requires (``kvweaver/backend.py:135-150``).
    """
    c_p = _through_origin(prefill)
    c_a = _through_origin(denoise)
    pts = [(m, us / k) for k, m, us in decode]
    if len({m for m, _ in pts}) < 2:
        raise ValueError("decode samples need at least two distinct batch sizes")
    n = len(pts)
    mx = sum(m for m, _ in pts) / n
    my = sum(y for _, y in pts) / n
    slope = sum((m - mx) * (y - my) for m, y in pts) / sum((m - mx) ** 2 for m, _ in pts)
    base = my - slope * mx
    return CostModelParams(max(0, round(c_p)), max(0, round(c_a)), max(0, round(base)),
                           max(0, round(slope)), max(1.0, float(contention)))


def closed_form_speedup(params: CostModelParams, n_tokens: int, k: int, p_len: int, S: int) -> float:
    """Steady-state IsolatedSequential / Unified frame-time ratio, the closed form
    of tests/test_acceptance.py:129-133 (one arrival per frame, m = N / k)."""
    p = params.c_prefill_per_token * p_len
    a = S * params.c_denoise_per_step
    m = max(1, -(-n_tokens // k))
    t_uni = p + a + k * (params.c_decode_base + params.c_decode_per_request * m)
    t_iso = 2 * p + a + n_tokens * (params.c_decode_base + params.c_decode_per_request)
    return t_iso / t_uni


def measure_stage_samples(backend, n_cams=(0, 1, 2, 3), prompt=32, steps=(1, 5, 10), rows=(1, 2, 4, 8, 16),
                          k=5, reps=5):
    """CUDA-event stage timings on a GPU backend (Pi05Backend): prefill at
    P = 256 * cams + prompt, denoise at S steps, decode of k tokens for m rows."""
    import torch

    from .kv_manager import BatchedState
    from .pi05 import Pi05Observation, synthetic_images

    def timed(fn):
        for _ in range(3):  # eager, graph capture, replay
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e3 / reps

    def obs(cams, seed):
        return Pi05Observation(tuple(range(100 + seed, 100 + seed + prompt)), 0,
                               synthetic_images(cams, seed) if cams else None)

    out = {"prefill": [], "denoise": [], "decode": []}
    for cams in n_cams:
        out["prefill"].append((256 * cams + prompt, timed(lambda: backend.prefill(obs(cams, 5)))))
    kv = backend.prefill(obs(n_cams[-1], 5))
    for s in steps:
        out["denoise"].append((s, timed(lambda: backend.action_denoise(kv, s))))
    kvs = [backend.prefill(obs(n_cams[-1], 7 + i)) for i in range(max(rows))]
    for m in rows:
        st = BatchedState(tuple(kvs[:m]), ((),) * m, (False,) * m, tuple(range(m)), (10 ** 6,) * m, (0,) * m)
        out["decode"].append((k, m, timed(lambda: backend.batched_language_decode(st, k))))
    return out
