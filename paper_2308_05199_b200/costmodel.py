"""Analytic timing model of the collectives, with B200-fitted constants
(mirror of gzccl.costmodel, /root/reference/pkg/src/gzccl/costmodel.py:31-158,
and of the clock-only timelines behind ``predicted_makespan``,
collectives.py:580-728).

The model is the reference's: alpha-beta messages, kernels costing
``launch + max(bytes, saturation) / throughput``, optional host staging,
compute/communication overlap and multi-stream batching.  The reference ships
placeholder numbers; :func:`b200_cost_params` loads constants fitted from
measurements of THIS implementation on B200 (``tools/calibrate_costmodel.py``
writes ``profiles/b200_cost_params.json``): the codec kernels' launch floor,
saturation size and throughput, the fused reduce step's extra cost, the
NVLink pull latency / bandwidth between two GPUs and the pinned host link.
With those, ``predicted_makespan("ring-allreduce", S, N)`` predicts the
measured one-process-per-GPU allreduce (checked in the calibration run).
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, fields

KERNEL_KINDS = ("compress", "decompress", "reduce")
DEFAULT_ASSUMED_CR = 64.0  # costmodel.py:27
_FITTED = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "b200_cost_params.json")


@dataclass(frozen=True)
class CostParams:
    """Link, kernel and behaviour parameters (costmodel.py:31-62); defaults
    are the reference's placeholders, :func:`b200_cost_params` the fit."""

    alpha: float = 1e-5
    beta: float = 8e-11
    launch: float = 1.5e-4
    saturation: float = 5.05e6
    compress_throughput: float = 1.28e11
    decompress_throughput: float = 1.28e11
    reduce_throughput: float = 4e11
    host_device_bandwidth: float = 2.4e10
    staging: bool = False
    overlap: bool = False
    multi_stream: bool = False

    def __post_init__(self):
        for f in fields(self):
            if f.type in ("bool", bool):
                continue
            v = getattr(self, f.name)
            if not (isinstance(v, (int, float)) and not isinstance(v, bool) and math.isfinite(v) and v > 0):
                raise ValueError(f"{f.name} must be a positive finite number, got {v!r}")

    def _rate(self, kind: str) -> float:
        if kind not in KERNEL_KINDS:
            raise ValueError(f"unknown kernel kind {kind!r}, expected one of {KERNEL_KINDS}")
        return getattr(self, kind + "_throughput")

    def msg_time(self, nbytes: float) -> float:
        """alpha + bytes * beta (costmodel.py:64-68)."""
        if nbytes < 0:
            raise ValueError("message size must be non-negative")
        return self.alpha + nbytes * self.beta

    def kernel_time(self, nbytes: float, kind: str) -> float:
        """launch + max(bytes, saturation) / throughput (costmodel.py:70-74)."""
        if nbytes < 0:
            raise ValueError("kernel size must be non-negative")
        return self.launch + max(nbytes, self.saturation) / self._rate(kind)

    def multi_launch_time(self, sizes, kind: str) -> float:
        """A batch of blocks: one launch over the sum with multi-stream batching,
        back-to-back kernels otherwise (costmodel.py:76-88)."""
        sizes = list(sizes)
        if not sizes:
            raise ValueError("multi_launch_time needs at least one block size")
        if self.multi_stream:
            return self.launch + max(sum(sizes), self.saturation) / self._rate(kind)
        return sum(self.kernel_time(b, kind) for b in sizes)

    def staging_time(self, nbytes: float) -> float:
        """Host round trip of a staged message (costmodel.py:90-96)."""
        if nbytes < 0:
            raise ValueError("staged size must be non-negative")
        return 2.0 * nbytes / self.host_device_bandwidth if self.staging else 0.0

    def step_time(self, comm_seconds: float, compute_seconds: float) -> float:
        """max (overlap) or sum of one step's sides (costmodel.py:98-104)."""
        if comm_seconds < 0 or compute_seconds < 0:
            raise ValueError("step components must be non-negative")
        return max(comm_seconds, compute_seconds) if self.overlap else comm_seconds + compute_seconds

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_dict(cls, d: dict) -> "CostParams":
        unknown = set(d) - {f.name for f in fields(cls)}
        if unknown:
            raise ValueError(f"unknown cost parameter(s): {sorted(unknown)}")
        return cls(**d)


def load_cost_params(path=None, **overrides) -> CostParams:
    """JSON file of parameters (missing fields keep their defaults) plus overrides (costmodel.py:117-134)."""
    d: dict = {}
    if path is not None:
        with open(path, "r", encoding="utf-8") as fh:
            loaded = json.load(fh)
        if not isinstance(loaded, dict):
            raise ValueError(f"cost config {path} must hold a JSON object")
        d.update(loaded)
    d.update(overrides)
    return CostParams.from_dict(d)


def b200_cost_params(path: str | None = None) -> CostParams:
    """The constants fitted on B200 by tools/calibrate_costmodel.py."""
    p = path or _FITTED
    with open(p, "r", encoding="utf-8") as fh:
        d = json.load(fh)
    return CostParams.from_dict(d["params"] if "params" in d else d)


# ---------------------------------------------------------------------------
# clock-only timelines (collectives.py:580-728): the step accounting of the
# simulated collectives without data
# ---------------------------------------------------------------------------


class _Costs:
    """Per-call constants of one timeline: kernel and message times."""

    def __init__(self, p: CostParams, kernel_bytes: float, msg: float, compressed: bool):
        self.p = p
        self.c = p.kernel_time(kernel_bytes, "compress") if compressed else 0.0
        self.d = p.kernel_time(kernel_bytes, "decompress") if compressed else 0.0
        self.r = p.kernel_time(kernel_bytes, "reduce")
        self.st = p.staging_time(msg)
        self.mt = p.msg_time(msg)

    def step(self, comm: float, compute: float) -> float:
        return self.p.step_time(comm, compute)


def _span_allgather(p, chunk, N, msg, compressed):  # _ring_allgather: compress once, decode every receipt
    if N < 2:
        return 0.0
    k = _Costs(p, chunk, msg, compressed)
    return k.step(k.st + k.mt, k.c + k.d) + (N - 2) * k.step(k.st + k.mt, k.d)


def _span_reduce_scatter(p, chunk, N, msg, compressed):  # N-1 steps of encode + decode + reduce
    if N < 2:
        return 0.0
    k = _Costs(p, chunk, msg, compressed)
    return (N - 1) * k.step(k.st + k.mt, k.c + k.d + k.r)


def _span_cprp2p(p, chunk, N, msg, compressed):  # N-1 hops of encode + decode
    if N < 2:
        return 0.0
    k = _Costs(p, chunk, msg, compressed)
    return (N - 1) * k.step(k.st + k.mt, k.c + k.d)


def _span_rd(p, nbytes, N, msg, compressed):
    """Per-rank clocks of rd_allreduce_c (collectives.py:349-424)."""
    if N < 2:
        return 0.0
    from .collectives import rd_plan

    pof2, r, steps, role, remapped, actual = rd_plan(N)
    k = _Costs(p, nbytes, msg, compressed)
    pre = 0.0 if p.overlap else k.c
    join = max if p.overlap else (lambda a, b: a + b)
    clock = [0.0] * N
    donors = list(range(0, 2 * r, 2))
    if r:
        for i in donors:  # donors post at clock 0
            clock[i] += k.step(k.st, k.c)
        wait = max(0.0, pre + k.st + k.mt)
        for i in donors:
            clock[i + 1] += k.step(wait, k.d + k.r)
    parts = [i for i in range(N) if role(i) != "donor"]
    for t in range(steps):
        snap = list(clock)
        for i in parts:
            j = actual(remapped(i) ^ (1 << t))
            wait = max(0.0, (snap[j] + pre + k.st + k.mt) - (snap[i] + pre + k.st))
            clock[i] = snap[i] + join(wait + k.st, k.c + k.d + k.r)
    if r:
        arrive = {i: clock[i + 1] + pre + k.st + k.mt for i in donors}
        for i in donors:
            clock[i + 1] += k.step(k.st, k.c)
        for i in donors:
            clock[i] = clock[i] + join(max(0.0, arrive[i] - clock[i]), k.d)
    return float(max(clock))


def _span_scatter(p, block, N, block_msg, compressed):
    """Tree arrival times of binomial_scatter_c (collectives.py:467-532)."""
    if N < 2:
        return 0.0
    from .collectives import scatter_children, scatter_msg_overhead

    t_mc = p.multi_launch_time([block] * N, "compress") if compressed else 0.0
    t_d = p.kernel_time(block, "decompress") if compressed else 0.0
    head = scatter_msg_overhead(N)
    arrival = [0.0] * N
    clock = [0.0] * N

    def forward(node: int, t0: float) -> float:
        staged = 0.0
        for child, lo, hi in scatter_children(node, N)[1]:
            mb = head + (hi - lo) * block_msg
            arrival[child] = t0 + staged + p.staging_time(mb) + p.msg_time(mb)
            staged += p.staging_time(mb)
        return staged

    staged = forward(0, 0.0 if p.overlap else t_mc)
    clock[0] = p.step_time(staged, t_mc)
    for vr in range(1, N):
        staged = forward(vr, arrival[vr])
        clock[vr] = p.step_time(arrival[vr] + staged, t_d)
    return max(clock)


_TIMELINES = {
    "ring-allgather": lambda p, D, N, cr, z: _span_allgather(p, D / N, N, D / N / cr, z),
    "lossless-allgather": lambda p, D, N, cr, z: _span_allgather(p, D / N, N, D / N / cr, z),
    "cprp2p-allgather": lambda p, D, N, cr, z: _span_cprp2p(p, D / N, N, D / N / cr, z),
    "ring-reduce-scatter": lambda p, D, N, cr, z: _span_reduce_scatter(p, D / N, N, D / N / cr, z),
    "lossless-reduce-scatter": lambda p, D, N, cr, z: _span_reduce_scatter(p, D / N, N, D / N / cr, z),
    "ring-allreduce": lambda p, D, N, cr, z: (_span_reduce_scatter(p, D / N, N, D / N / cr, z)
                                              + _span_allgather(p, D / N, N, D / N / cr, z)),
    "lossless-allreduce": lambda p, D, N, cr, z: (_span_reduce_scatter(p, D / N, N, D / N / cr, z)
                                                  + _span_allgather(p, D / N, N, D / N / cr, z)),
    "rd-allreduce": lambda p, D, N, cr, z: _span_rd(p, D, N, D / cr, z),
    "binomial-scatter": lambda p, D, N, cr, z: _span_scatter(p, D / N, N, D / N / cr, z),
    "lossless-scatter": lambda p, D, N, cr, z: _span_scatter(p, D / N, N, D / N / cr, z),
}


def predicted_makespan(algorithm: str, data_bytes: float, ranks: int, params: CostParams | None = None,
                       assumed_cr: float = DEFAULT_ASSUMED_CR) -> float:
    """Modelled makespan without data (collectives.py:688-728): data_bytes is the
    per-rank buffer of the reductions and the total size of allgather/scatter;
    messages are raw / assumed_cr (1 for the lossless twins)."""
    from .collectives import get_algorithm

    p = params if params is not None else CostParams()
    if ranks < 1:
        raise ValueError("ranks must be >= 1")
    if data_bytes <= 0:
        raise ValueError("data_bytes must be positive")
    if assumed_cr <= 0:
        raise ValueError("assumed_cr must be positive")
    info = get_algorithm(algorithm)
    fn = _TIMELINES.get(algorithm)
    if fn is None:
        raise ValueError(f"no analytic timeline for {algorithm!r}")
    compressed = not info.lossless
    return fn(p, float(data_bytes), ranks, assumed_cr if compressed else 1.0, compressed)
