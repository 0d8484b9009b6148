"""Per-rank step plans of the compressed collectives (pure Python, no device).

The plans restate the reference schedules (collectives.py:215-308, 449-532)
for ONE rank of a real communicator, in the fused form the device path runs:
the chunk rank i compresses at reduce-scatter step s+1 is exactly the chunk it
reduced at step s (collectives.py:274-290), so every step after the first is
a single "reduce" = compress(op(local, decompress(recv))).

The same plans drive the GPU executor (comm.py, NVLink peer memory) and the
CPU gloo executor used by the multi-process tests, so the schedule logic is
tested without a GPU.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Compress:
    """Compress local chunk `chunk` and deliver it to `dst`'s RS slot `slot`."""

    chunk: int
    dst: int
    slot: int


@dataclass(frozen=True)
class Reduce:
    """Wait for RS slot `slot`, combine with local chunk `chunk`, compress.

    last=False: deliver the new blob to `dst`'s slot `slot + 1`.
    last=True : this is the owned chunk: keep the f32 result (exact) and the
                blob, which the allgather serves to every other rank.
    """

    slot: int
    chunk: int
    dst: int
    last: bool


@dataclass(frozen=True)
class Gather:
    """Decode owner `owner`'s compress-once blob into output chunk `chunk`."""

    owner: int
    chunk: int


def ring_allreduce_plan(N: int, i: int) -> list:
    """ring_allreduce_c (collectives.py:294-308) for rank i of N."""
    if N == 1:
        return []
    right = (i + 1) % N
    plan = [Compress(chunk=i, dst=right, slot=0)]
    for s in range(N - 1):
        c_in = (i - s - 1) % N  # collectives.py:287
        last = s == N - 2
        plan.append(Reduce(slot=s, chunk=c_in, dst=i if last else right, last=last))
    for k in range(1, N):
        j = (i - k) % N  # arrival order of the reference ring (collectives.py:240-241)
        plan.append(Gather(owner=j, chunk=(j + 1) % N))
    return plan


def owned_chunk(N: int, i: int) -> int:
    """Chunk whose fully reduced value rank i holds after the reduce-scatter (collectives.py:291)."""
    return (i + 1) % N


def ring_reduce_scatter_plan(N: int, i: int) -> list:
    """ring_reduce_scatter_c (collectives.py:258-291): the allreduce plan minus the allgather."""
    return [p for p in ring_allreduce_plan(N, i) if not isinstance(p, Gather)]


def scatter_route(N: int, root: int = 0):
    """(parent, own_vr, [(child, lo, hi), ...]) per actual rank of the binomial tree.

    Virtual rank vr = (rank - root) mod N (collectives.py:496); message ranges
    are virtual block indices (collectives.py:449-464).
    """
    from .collectives import scatter_children

    routes = {}
    order = [(root + j) % N for j in range(N)]
    for vr in range(N):
        extent, sends = scatter_children(vr, N)
        parent = None if vr == 0 else order[vr - extent]
        routes[order[vr]] = (parent, vr, [(order[c], lo, hi) for c, lo, hi in sends])
    return routes


# ---------------------------------------------------------------------------
# recursive doubling (collectives.py:349-424, RecursiveDoublingPlan 48-86)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class RdSend:
    """Send message number `k` to `dst`.  src is None: the message is
    compress(data).  Otherwise first data = op(data, decompress(src's message
    k_in)) and the message is compress(data) -- one fused kernel."""

    k: int
    dst: int
    src: int | None = None
    k_in: int | None = None


@dataclass(frozen=True)
class RdRecvLast:
    """data = op(data, decompress(src's message k_in)) (reduce) or
    data = decompress(...) (a donor receiving its absorber's result)."""

    src: int
    k_in: int
    reduce: bool


def rd_allreduce_plan(N: int, i: int) -> list:
    """rd_allreduce_c for rank i of N, in fused form.  Message numbers: 0 = a
    donor's buffer, 1..steps = the exchange steps, steps+1 = an absorber's
    final result sent back to its donor (collectives.py:381-435)."""
    if N == 1:
        return []
    pof2 = 1 << (N.bit_length() - 1)
    r = N - pof2
    steps = pof2.bit_length() - 1
    K = steps + 2

    def role(j):
        return ("donor" if j % 2 == 0 else "absorber") if j < 2 * r else "direct"

    def remapped(j):
        return j // 2 if role(j) == "absorber" else j - r

    def actual(v):
        return 2 * v + 1 if v < r else v + r

    if role(i) == "donor":  # 381-386, 430-435
        return [RdSend(k=0, dst=i + 1), RdRecvLast(src=i + 1, k_in=K - 1, reduce=False)]
    part = [actual(remapped(i) ^ (1 << t)) for t in range(steps)]
    plan = []
    if role(i) == "absorber":  # 389-397: the donor folded in, fused with the step-0 compression
        plan.append(RdSend(k=1, dst=part[0], src=i - 1, k_in=0))
    else:
        plan.append(RdSend(k=1, dst=part[0]))
    for t in range(steps):  # 399-418
        if t + 1 < steps:
            plan.append(RdSend(k=t + 2, dst=part[t + 1], src=part[t], k_in=t + 1))
        elif role(i) == "absorber":  # 420-427: the result goes back to the donor
            plan.append(RdSend(k=K - 1, dst=i - 1, src=part[t], k_in=t + 1))
        else:
            plan.append(RdRecvLast(src=part[t], k_in=t + 1, reduce=True))
    return plan
