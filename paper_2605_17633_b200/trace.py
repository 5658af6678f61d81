"""Per-kernel CUDA-event tracing (the reference's per-block wall clock, encoder.py:342,372,
made device-side).

``Tracer.span(name, flops=, bytes=)`` records an event pair on the launching
(current) stream around one native launch, with the launch's ALGORITHMIC work
(skipped tiles / rows not counted).  Events are asynchronous, so tracing the
timed region costs a few host microseconds per launch and no device sync;
``summary()`` synchronises once and aggregates time, launches, FLOPs and
bytes per kernel name.
"""

from __future__ import annotations

from collections import defaultdict
from contextlib import contextmanager

import torch


class Tracer:
    def __init__(self):
        self.records: list = []

    @contextmanager
    def span(self, name: str, flops: float = 0.0, bytes: float = 0.0):  # noqa: A002
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        yield
        e.record()
        self.records.append((name, s, e, flops, bytes))

    def reset(self):
        self.records.clear()

    def summary(self) -> dict:
        torch.cuda.synchronize()
        agg = defaultdict(lambda: dict(ms=0.0, launches=0, flops=0.0, bytes=0.0))
        for name, s, e, f, b in self.records:
            a = agg[name]
            a["ms"] += s.elapsed_time(e)
            a["launches"] += 1
            a["flops"] += _resolve(f)
            a["bytes"] += _resolve(b)
        return dict(agg)


def _resolve(v) -> float:
    """Work is a number, or (device count tensor, per-item work) resolved after the sync."""
    if isinstance(v, tuple):
        n, per = v
        return float(n.item()) * per
    return float(v)


class _Null:
    @contextmanager
    def span(self, *a, **k):
        yield


NULL = _Null()
