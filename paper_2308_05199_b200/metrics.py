"""Accuracy statistics and the collective report (mirror of gzccl.metrics,
/root/reference/pkg/src/gzccl/metrics.py).

Same names, fields, formulas and ``to_dict`` schema ("gzccl.report.v1") as the
reference, so code that consumes a reference report reads ours unchanged.
The statistics are computed on the device in binary64 when given CUDA tensors
(numpy arrays are accepted too); reductions are summed in a different order
than numpy's pairwise sums, so mse / mean agree to ~1e-15 relative, max |err|
exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch


def _f64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().reshape(-1).to(torch.float64)
    return torch.from_numpy(np.asarray(a, dtype=np.float64).reshape(-1))


def _pair(ref, test) -> tuple[torch.Tensor, torch.Tensor]:
    r, t = _f64(ref), _f64(test)
    if r.shape != t.shape:
        raise ValueError(f"length mismatch: {tuple(r.shape)} vs {tuple(t.shape)}")  # metrics.py:14-15
    if r.device != t.device:
        t = t.to(r.device)
    return r, t


def max_abs_error(ref, test) -> float:
    """Largest elementwise |ref - test|; 0 for empty buffers (metrics.py:11-20)."""
    r, t = _pair(ref, test)
    return 0.0 if r.numel() == 0 else float((r - t).abs().max())


def mean_signed_error(ref, test) -> float:
    """Mean of (test - ref) (metrics.py:23-32)."""
    r, t = _pair(ref, test)
    return 0.0 if r.numel() == 0 else float((t - r).mean())


def mse(ref, test) -> float:
    r, t = _pair(ref, test)
    return 0.0 if r.numel() == 0 else float(((r - t) ** 2).mean())


def psnr(ref, test) -> float:
    """10 log10(range^2 / mse), range = max(ref) - min(ref) (metrics.py:45-62)."""
    r, t = _pair(ref, test)
    if r.numel() == 0:
        raise ValueError("psnr needs non-empty buffers")
    err = float(((r - t) ** 2).mean())
    if err == 0.0:
        return math.inf
    rng = float(r.max() - r.min())
    if rng == 0.0:
        raise ValueError("psnr undefined: zero reference range with nonzero error")
    return 10.0 * math.log10(rng * rng / err)


def compression_ratio(original_bytes: float, compressed_bytes: float) -> float:
    if compressed_bytes <= 0:
        raise ValueError("compressed size must be positive")
    return float(original_bytes) / float(compressed_bytes)


@dataclass(frozen=True)
class AccuracyStats:
    """Error statistics of a collective's outputs against its lossless rerun (metrics.py:71-102)."""

    max_abs_err: float
    mse: float
    psnr: float  # dB; +inf when the outputs equal the lossless rerun
    mean_signed_err: float

    @classmethod
    def of(cls, ref, test) -> "AccuracyStats":
        r, t = _pair(ref, test)
        if r.numel() == 0:
            return cls(0.0, 0.0, math.inf, 0.0)
        d = t - r
        err = float((d * d).mean())
        if err == 0.0:
            db = math.inf
        else:
            rng = float(r.max() - r.min())
            db = 10.0 * math.log10(rng * rng / err) if rng > 0 else -math.inf
        return cls(max_abs_err=float(d.abs().max()), mse=err, psnr=db, mean_signed_err=float(d.mean()))

    def to_dict(self) -> dict:
        return {
            "max_abs_err": self.max_abs_err,
            "mse": self.mse,
            "psnr_db": "inf" if math.isinf(self.psnr) and self.psnr > 0 else self.psnr,
            "mean_signed_err": self.mean_signed_err,
        }


_BUCKETS = (("compression", ("compress", "decompress")), ("communication", ("comm",)),
            ("reduction", ("reduce",)), ("others", ("staging", "other")))


def phase_breakdown(phase_seconds: dict) -> dict:
    """Percent of the phase time per bucket, summing to 100; no time at all
    counts as 100 % others (metrics.py:105-127)."""
    secs = {b: sum(phase_seconds.get(k, 0.0) for k in keys) for b, keys in _BUCKETS}
    total = sum(secs.values())
    if total <= 0.0:
        return {b: (100.0 if b == "others" else 0.0) for b, _ in _BUCKETS}
    return {b: 100.0 * v / total for b, v in secs.items()}


@dataclass(frozen=True)
class CollectiveReport:
    """Everything a collective run produced besides its outputs (metrics.py:130-180).

    On this implementation ``phase_seconds`` are MEASURED device seconds per
    kernel kind (CUDA events; the fused reduce step counts as "reduce") and
    ``makespan_seconds`` is the measured device time of the whole run with
    all ranks on one GPU; ``extra["predicted_makespan_b200"]`` is the cost
    model (costmodel.py) with B200-fitted constants for the one-process-per-GPU
    execution.
    """

    algorithm: str
    ranks: int
    root: int
    elements_per_rank: int | None
    total_elements: int
    eb: float | None
    codec: str
    reduce_op: str | None
    counters: dict
    counters_per_rank: list
    phase_seconds: dict
    makespan_seconds: float
    accuracy: AccuracyStats
    compression_ratio: float | None
    flags: dict
    seed: int | None = None
    data_source: str | None = None
    extra: dict = field(default_factory=dict)

    @property
    def breakdown_pct(self) -> dict:
        return phase_breakdown(self.phase_seconds)

    # key order of the reference's report schema (metrics.py:158-180)
    _KEYS = ("algorithm", "ranks", "root", "elements_per_rank", "total_elements", "eb", "codec", "reduce_op",
             "seed", "data_source", "flags", "counters", "counters_per_rank", "phase_seconds", "breakdown_pct",
             "makespan_seconds", "accuracy", "compression_ratio")

    def to_dict(self) -> dict:
        d = {"schema": "gzccl.report.v1"}
        for k in self._KEYS:
            v = getattr(self, k)
            if k == "accuracy":
                v = v.to_dict()
            elif k == "counters_per_rank":
                v = [dict(c) for c in v]
            elif isinstance(v, dict):
                v = dict(v)
            d[k] = v
        d.update(self.extra)
        return d
