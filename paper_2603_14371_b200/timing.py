"""CUDA-event stage timing for the measured-latency backends.

The reference prices latency with an integer-us cost model
(``kvweaver/backend.py:170-177``; its toy prices are zero).  The B200
backends instead record CUDA events on the launching stream around each
stage and the scheduler reads them once per frame (``scheduler._stage``),
so a FrameTrace carries measured device microseconds in the same fields.
"""

from __future__ import annotations

import contextlib


class StageMeter:
    def __init__(self):
        self._spans: dict[str, list] = {}
        self._extra: dict[str, float] = {}
        self._open: dict[str, object] = {}

    @contextlib.contextmanager
    def span(self, stage: str):
        import torch
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            self._spans.setdefault(stage, []).append((s, e))

    def begin(self, stage: str) -> None:
        import torch
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        self._open[stage] = s

    def end(self, stage: str) -> None:
        import torch
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self._spans.setdefault(stage, []).append((self._open.pop(stage), e))

    def put(self, stage: str, us: float) -> None:
        """Add a duration timed elsewhere (e.g. on the action-expert lane)."""
        self._extra[stage] = self._extra.get(stage, 0.0) + us

    def take(self, stage: str) -> int:
        spans = self._spans.pop(stage, [])
        extra = self._extra.pop(stage, 0.0)
        if spans:
            spans[-1][1].synchronize()
        return int(round(sum(s.elapsed_time(e) for s, e in spans) * 1000.0 + extra))

    def clear(self) -> None:
        self._spans.clear()
        self._extra.clear()
        self._open.clear()
