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

    def take(self, stage: str) -> int:
        spans = self._spans.pop(stage, [])
        if not spans:
            return 0
        spans[-1][1].synchronize()
        return int(round(sum(s.elapsed_time(e) for s, e in spans) * 1000.0))

    def clear(self) -> None:
        self._spans.clear()
