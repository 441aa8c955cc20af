"""Robot-stream sharding across GPUs.

Streams are independent: stream s runs on rank s mod world, each rank owns a
full replica of the weights, its own KV pool, manager and CUDA graphs.  The
only cross-rank traffic is end-of-run metric reduction (max elapsed time, sum
of actions / tokens), done with torch.distributed (NCCL on GPUs, gloo in the
CPU tests) — never on the per-frame path.
"""

from __future__ import annotations

__all__ = ["streams_for_rank", "reduce_metrics"]


def streams_for_rank(total_streams: int, world: int, rank: int) -> list[int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return [s for s in range(total_streams) if s % world == rank]


def reduce_metrics(elapsed_s: float, actions: int, tokens: int, streams: int, h: int,
                   device: str = "cpu") -> dict:
    """Whole-job aggregates: time is the max over ranks, counts are sums."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([elapsed_s], dtype=torch.float64, device=device)
    c = torch.tensor([actions, tokens, streams], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    sec = t.item()
    a, k, s = (int(v) for v in c.tolist())
    return {"elapsed_s": sec, "actions": a, "tokens": k, "streams": s,
            "action_hz": h * a / sec if sec else 0.0,
            "action_hz_per_stream": h * a / sec / s if sec and s else 0.0,
            "tok_s_per_stream": k / sec / s if sec and s else 0.0}
