"""Compression-enabled collectives: schedules over the device codec.

The reference (``/root/reference/pkg/src/gzccl/collectives.py``) runs every
rank in one process over a simulated network.  This module keeps its
algorithm ids, schedules and per-rank outputs and provides two drivers:

* ``*_virtual`` / :func:`run_collective`: all N ranks on ONE GPU in one
  process, executing the reference's two-pass step schedule with the device
  kernels.  Used for parity (every message is byte-comparable to the
  reference trace) and on single-GPU boxes.
* :mod:`paper_2308_05199_b200.comm`: one process per GPU, blobs moved over
  NVLink peer memory (CUDA IPC) by the kernels themselves.

Key fusion (collectives.py:274-290): the chunk rank i compresses at RS step
s+1 is exactly the chunk it reduced at step s, so each RS step is ONE kernel
``compress(op(local, decompress(recv)))`` (csrc gz_reduce_step).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .codec import BLOCK, DeviceBlob, Workspace, _check_eb, _NONE, _stream, compress, decompress

REDUCE_OPS = ("sum", "max")  # collectives.py:27
_OP_CODE = {"sum": 0, "max": 1}


def chunk_spans(n: int, ranks: int) -> list[tuple[int, int]]:
    """Partition [0, n) into ``ranks`` chunks of ceil(n/ranks) (collectives.py:42-45)."""
    step = -(-n // ranks) if n else 0
    return [(min(c * step, n), min((c + 1) * step, n)) for c in range(ranks)]


def _check_op(op: str) -> int:
    if op not in _OP_CODE:
        raise ValueError(f"unknown reduce op {op!r}, expected one of {REDUCE_OPS}")
    return _OP_CODE[op]


@dataclass
class Counters:
    """Per-rank operation counts (simnet.OpCounters subset, simnet.py:50-74)."""

    n_compress: int = 0
    n_decompress: int = 0
    n_messages: int = 0
    bytes_sent: int = 0
    raw_bytes_in: int = 0
    blob_bytes_out: int = 0

    def as_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class Trace:
    """Messages as (src, dst, payload bytes), like Network(record_payloads=True)."""

    msgs: list = field(default_factory=list)

    def add(self, src: int, dst: int, blob) -> None:
        self.msgs.append((src, dst, bytes(blob)))


def reduce_step(recv: DeviceBlob, local: torch.Tensor, eb: float, op: str, ws: Workspace, acc_out=None,
                stream=None) -> DeviceBlob:
    """One fused RS step: compress(op(local, decompress(recv))) in one kernel."""
    lib = L.lib()
    m = local.numel()
    if recv.n != m:
        raise ValueError(f"reduce shape mismatch: ({m},) vs ({recv.n},)")  # collectives.py:33-34
    cap = int(lib.gz_compress_bound(m))
    out = torch.empty(cap, dtype=torch.uint8, device=local.device)
    sc = torch.empty(int(lib.gz_sidecar_bytes(m)), dtype=torch.uint8, device=local.device)
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(m)))
    L.check(lib.gz_reduce_step(recv.data.data_ptr(), recv.sidecar.data_ptr(), local.data_ptr(), m, float(eb),
                               _check_op(op), acc_out.data_ptr() if acc_out is not None else None, out.data_ptr(), cap,
                               ws.len_ptr(), sc.data_ptr(), tws.data_ptr(), tws.numel(), ws.status_ptr(),
                               _stream(stream)), "gz_reduce_step")
    st = ws.read_status(stream)
    return DeviceBlob(out[: int(st[4])], sc, m, float(eb))


def _dev_inputs(buffers, size: int, device) -> list[torch.Tensor]:
    if len(buffers) != size:
        raise ValueError(f"expected {size} per-rank buffers, got {len(buffers)}")  # collectives.py:202-205
    out = []
    for b in buffers:
        if isinstance(b, torch.Tensor):
            t = b.detach().to(device=device, dtype=torch.float32).reshape(-1).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(b, dtype="<f4").reshape(-1)).to(device)
        out.append(t)
    return out


def _require_equal(bufs) -> int:  # collectives.py:208-212
    lengths = {b.numel() for b in bufs}
    if len(lengths) > 1:
        raise ValueError(f"per-rank buffers must have equal length, got {sorted(lengths)}")
    return bufs[0].numel()


def _check_finite(bufs) -> None:
    for b in bufs:
        bad = (~torch.isfinite(b)).nonzero()
        if bad.numel():
            raise ValueError(f"non-finite value at offset {int(bad[0])}")


def ring_reduce_scatter_virtual(buffers, eb, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                                counters: list | None = None, _keep_blobs: bool = False):
    """ring_reduce_scatter_c (collectives.py:258-291) with N virtual ranks on one GPU.

    Returns the per-rank owned chunks (rank i owns chunk (i+1) mod N); with
    ``_keep_blobs`` also each rank's compressed owned chunk (the allgather's
    compress-once blob, produced by the last fused step).
    """
    ebf = _check_eb(eb)
    _check_op(op)
    ws = ws or Workspace()
    N = len(buffers)
    bufs = _dev_inputs(buffers, N, ws.device)
    n = _require_equal(bufs)
    _check_finite(bufs)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return ([bufs[0].clone()], [None]) if _keep_blobs else [bufs[0].clone()]
    spans = chunk_spans(n, N)

    def chunk(i, c):
        lo, hi = spans[c]
        return bufs[i][lo:hi]

    # step 0 sends: rank i compresses its own chunk i
    sending = []
    for i in range(N):
        blob = compress(chunk(i, i), ebf, ws)
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * blob.n
        counters[i].blob_bytes_out += len(blob)
        sending.append(blob)
    owned = [None] * N
    for s in range(N - 1):
        if trace is not None:
            for i in range(N):
                trace.add(i, (i + 1) % N, sending[i])
        for i in range(N):
            counters[i].n_messages += 1
            counters[i].bytes_sent += len(sending[i])
        nxt = []
        for i in range(N):
            recv = sending[(i - 1) % N]
            c_in = (i - s - 1) % N
            last = s == N - 2
            acc = torch.empty(spans[c_in][1] - spans[c_in][0], dtype=torch.float32, device=ws.device) if last else None
            blob = reduce_step(recv, chunk(i, c_in), ebf, op, ws, acc_out=acc)
            counters[i].n_decompress += 1
            if not last or _keep_blobs:
                counters[i].n_compress += 1
                counters[i].raw_bytes_in += 4 * blob.n
                counters[i].blob_bytes_out += len(blob)
            if last:
                owned[i] = acc
            nxt.append(blob)
        sending = nxt
    return (owned, sending) if _keep_blobs else owned


def _allgather_blobs(blobs, owned, chunk_of, ws: Workspace, trace: Trace | None, counters: list):
    """_ring_allgather (collectives.py:215-244): blobs compressed once, forwarded unchanged."""
    N = len(blobs)
    gathered = [{chunk_of(i): owned[i]} for i in range(N)]
    carry = list(blobs)
    for s in range(N - 1):
        if trace is not None:
            for i in range(N):
                trace.add(i, (i + 1) % N, carry[i])
        for i in range(N):
            counters[i].n_messages += 1
            counters[i].bytes_sent += len(carry[i])
        carry = [carry[(i - 1) % N] for i in range(N)]
        for i in range(N):
            gathered[i][chunk_of((i - 1 - s) % N)] = decompress(carry[i], ws)
            counters[i].n_decompress += 1
    return gathered


def ring_allreduce_virtual(buffers, eb, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                           counters: list | None = None) -> list[torch.Tensor]:
    """ring_allreduce_c (collectives.py:294-308): RS, then compress-once AG."""
    ws = ws or Workspace()
    N = len(buffers)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        bufs = _dev_inputs(buffers, 1, ws.device)
        _check_finite(bufs)
        return [bufs[0].clone()]
    owned, blobs = ring_reduce_scatter_virtual(buffers, eb, op, ws, trace, counters, _keep_blobs=True)
    gathered = _allgather_blobs(blobs, owned, lambda i: (i + 1) % N, ws, trace, counters)
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


def ring_allgather_virtual(chunks, eb, ws: Workspace | None = None, trace: Trace | None = None,
                           counters: list | None = None) -> list[torch.Tensor]:
    """ring_allgather_c (collectives.py:247-255), unequal chunk lengths allowed."""
    ebf = _check_eb(eb)
    ws = ws or Workspace()
    N = len(chunks)
    owned = _dev_inputs(chunks, N, ws.device)
    _check_finite(owned)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return [owned[0].clone()]
    blobs = []
    for i in range(N):
        blobs.append(compress(owned[i], ebf, ws))
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * owned[i].numel()
        counters[i].blob_bytes_out += len(blobs[-1])
    gathered = _allgather_blobs(blobs, owned, lambda i: i, ws, trace, counters)
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


def decompress_reduce(recv: DeviceBlob, local: torch.Tensor, eb: float, op: str, ws: Workspace, out=None,
                      stream=None) -> torch.Tensor:
    """op(local, decompress(recv)) in one kernel (no re-compression)."""
    m = local.numel()
    if recv.n != m:
        raise ValueError(f"reduce shape mismatch: ({m},) vs ({recv.n},)")  # collectives.py:33-34
    out = torch.empty_like(local) if out is None else out
    L.check(L.lib().gz_decompress_reduce(recv.data.data_ptr(), recv.sidecar.data_ptr(), local.data_ptr(), m, float(eb),
                                         _check_op(op), out.data_ptr(), ws.status_ptr(), _stream(stream)),
            "gz_decompress_reduce")
    return out


def rd_plan(N: int):
    """RecursiveDoublingPlan (collectives.py:48-86): pof2, r, steps and the
    role / remapped / actual maps (donors are the even ranks below 2r)."""
    pof2 = 1 << (N.bit_length() - 1)
    r = N - pof2
    steps = pof2.bit_length() - 1

    def role(i):
        return ("donor" if i % 2 == 0 else "absorber") if i < 2 * r else "direct"

    def remapped(i):
        if role(i) == "donor":
            raise ValueError(f"rank {i} is a donor and has no remapped id")
        return i // 2 if role(i) == "absorber" else i - r

    def actual(v):
        if not 0 <= v < pof2:
            raise ValueError(f"remapped id {v} out of range [0, {pof2})")
        return 2 * v + 1 if v < r else v + r

    return pof2, r, steps, role, remapped, actual


def rd_allreduce_virtual(buffers, eb, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                         counters: list | None = None) -> list[torch.Tensor]:
    """rd_allreduce_c (collectives.py:349-424) with N virtual ranks on one GPU.

    Whole-buffer exchanges.  The message a participant sends at step t+1 is
    compress(data after step t), so every reduction that is followed by a
    send is one fused kernel compress(op(data, decompress(recv))) that also
    updates data in place (gz_reduce_step); the last reduction of a rank
    that sends nothing more is gz_decompress_reduce.
    """
    ebf = _check_eb(eb)
    _check_op(op)
    ws = ws or Workspace()
    N = len(buffers)
    data = _dev_inputs(buffers, N, ws.device)
    _require_equal(data)
    _check_finite(data)
    data = [d.clone() for d in data]
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return data
    pof2, r, steps, role, remapped, actual = rd_plan(N)
    donors = [i for i in range(N) if role(i) == "donor"]
    parts = [i for i in range(N) if role(i) != "donor"]

    def send(i, dst, blob):
        if trace is not None:
            trace.add(i, dst, blob)
        counters[i].n_messages += 1
        counters[i].bytes_sent += len(blob)

    def comp(i):
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * data[i].numel()
        b = compress(data[i], ebf, ws)
        counters[i].blob_bytes_out += len(b)
        return b

    def fused(i, recv):  # data[i] = op(data[i], dec(recv)); returns compress(data[i])
        counters[i].n_decompress += 1
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * data[i].numel()
        b = reduce_step(recv, data[i], ebf, op, ws, acc_out=data[i])
        counters[i].blob_bytes_out += len(b)
        return b

    def last(i, recv):  # data[i] = op(data[i], dec(recv))
        counters[i].n_decompress += 1
        decompress_reduce(recv, data[i], ebf, op, ws, out=data[i])

    # message each participant sends at the next exchange step
    nxt = {}
    if r:
        dblob = {}
        for i in donors:  # 381-386
            dblob[i] = comp(i)
            send(i, i + 1, dblob[i])
        for i in parts:  # 389-397: absorbers fold their donor in; the fused kernel also
            # produces their step-0 message
            nxt[i] = fused(i, dblob[i - 1]) if role(i) == "absorber" else None
    for t in range(steps):  # 399-418
        msg = {}
        for i in parts:
            msg[i] = nxt[i] if nxt.get(i) is not None else comp(i)
            send(i, actual(remapped(i) ^ (1 << t)), msg[i])
        for i in parts:
            recv = msg[actual(remapped(i) ^ (1 << t))]
            more = t + 1 < steps or role(i) == "absorber"
            if more:
                nxt[i] = fused(i, recv)
            else:
                last(i, recv)
    if r:
        for i in parts:  # 420-427: the absorbers' final data, already compressed
            if role(i) == "absorber":
                send(i, i - 1, nxt[i])
        for i in donors:  # 430-435
            counters[i].n_decompress += 1
            data[i] = decompress(nxt[i + 1], ws)
    return data


# ---------------------------------------------------------------------------
# comparators (collectives.py:311-341, 545-566)
# ---------------------------------------------------------------------------


def cprp2p_allgather_virtual(chunks, eb, ws: Workspace | None = None, trace: Trace | None = None,
                             counters: list | None = None) -> list[torch.Tensor]:
    """cprp2p_allgather (collectives.py:311-341): the compress-per-hop baseline;
    every hop decompresses and re-compresses, so a chunk that travelled h hops
    carries up to h * eb of error (N-1 compressions and decompressions per rank)."""
    ebf = _check_eb(eb)
    ws = ws or Workspace()
    N = len(chunks)
    owned = _dev_inputs(chunks, N, ws.device)
    _check_finite(owned)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return [owned[0].clone()]
    gathered = [{i: owned[i]} for i in range(N)]
    current = list(owned)
    for s in range(N - 1):
        sent = []
        for i in range(N):
            b = compress(current[i], ebf, ws)
            counters[i].n_compress += 1
            counters[i].raw_bytes_in += 4 * current[i].numel()
            counters[i].blob_bytes_out += len(b)
            sent.append(b)
            if trace is not None:
                trace.add(i, (i + 1) % N, b)
            counters[i].n_messages += 1
            counters[i].bytes_sent += len(b)
        for i in range(N):
            vals = decompress(sent[(i - 1) % N], ws)
            counters[i].n_decompress += 1
            gathered[i][(i - 1 - s) % N] = vals
            current[i] = vals
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


def _raw_op(op: str, local: torch.Tensor, received: torch.Tensor) -> torch.Tensor:
    # _apply_op (collectives.py:32-39) on verbatim f32 payloads
    if op == "sum":
        return local + received
    return torch.where(torch.isnan(local) | (local > received), local, received)  # np.maximum(local, received)


def _raw_send(trace, counters, i, dst, t: torch.Tensor):
    if trace is not None:
        trace.add(i, dst, t.detach().cpu().numpy().astype("<f4").tobytes())
    counters[i].n_messages += 1
    counters[i].bytes_sent += 4 * t.numel()


def lossless_ring_reduce_scatter(buffers, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                                 counters: list | None = None):
    """ring_reduce_scatter_c with the RawTransport (the "lossless-*" twins,
    collectives.py:94-111, 560-566): verbatim f32 messages, no codec."""
    _check_op(op)
    ws = ws or Workspace()
    N = len(buffers)
    bufs = _dev_inputs(buffers, N, ws.device)
    n = _require_equal(bufs)
    _check_finite(bufs)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return [bufs[0].clone()]
    spans = chunk_spans(n, N)
    acc = [[b[lo:hi].clone() for lo, hi in spans] for b in bufs]
    for s in range(N - 1):
        sent = [acc[i][(i - s) % N] for i in range(N)]
        for i in range(N):
            _raw_send(trace, counters, i, (i + 1) % N, sent[i])
        sent = [t.clone() for t in sent]
        for i in range(N):
            c_in = (i - s - 1) % N
            acc[i][c_in] = _raw_op(op, acc[i][c_in], sent[(i - 1) % N])
    return [acc[i][(i + 1) % N] for i in range(N)]


def _lossless_allgather_owned(owned, chunk_of, trace, counters):
    N = len(owned)
    gathered = [{chunk_of(i): owned[i]} for i in range(N)]
    carry = list(owned)
    for s in range(N - 1):
        for i in range(N):
            _raw_send(trace, counters, i, (i + 1) % N, carry[i])
        carry = [carry[(i - 1) % N] for i in range(N)]
        for i in range(N):
            gathered[i][chunk_of((i - 1 - s) % N)] = carry[i].clone()
    return gathered


def lossless_ring_allgather(chunks, ws: Workspace | None = None, trace: Trace | None = None,
                            counters: list | None = None):
    ws = ws or Workspace()
    N = len(chunks)
    owned = _dev_inputs(chunks, N, ws.device)
    _check_finite(owned)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    if N == 1:
        return [owned[0].clone()]
    g = _lossless_allgather_owned(owned, lambda i: i, trace, counters)
    return [torch.cat([g[i][c] for c in range(N)]) for i in range(N)]


def lossless_ring_allreduce(buffers, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                            counters: list | None = None):
    ws = ws or Workspace()
    N = len(buffers)
    if counters is None:
        counters = [Counters() for _ in range(N)]
    owned = lossless_ring_reduce_scatter(buffers, op, ws, trace, counters)
    if N == 1:
        return owned
    g = _lossless_allgather_owned(owned, lambda i: (i + 1) % N, trace, counters)
    return [torch.cat([g[i][c] for c in range(N)]) for i in range(N)]


def lossless_binomial_scatter(root_data, N: int, counts=None, root: int = 0, ws: Workspace | None = None):
    """binomial_scatter_c with the RawTransport: every rank gets its slice verbatim."""
    ws = ws or Workspace()
    x = _dev_inputs([root_data], 1, ws.device)[0]
    _check_finite([x])
    counts = scatter_counts(x.numel(), N, counts)
    lo = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return [x[lo[r]:lo[r + 1]].clone() for r in range(N)]


# ---------------------------------------------------------------------------
# binomial-tree scatter (collectives.py:432-532)
# ---------------------------------------------------------------------------

_SC_HDR_BYTES = 24  # "<QQQ": block count, first block, one-past-last block


def scatter_msg_overhead(ranks: int) -> int:
    """Bytes of table metadata carried by every scatter message (collectives.py:444-446)."""
    return _SC_HDR_BYTES + 8 * ranks


def scatter_children(vr: int, size: int):
    """Receive extent and (child, lo, hi) sends of one tree node (collectives.py:449-464)."""
    mask = 1
    while mask < size:
        if vr & mask:
            break
        mask <<= 1
    extent = mask
    sends = []
    mask >>= 1
    while mask:
        child = vr + mask
        if child < size:
            sends.append((child, child, min(child + mask, size)))
        mask >>= 1
    return extent, sends


def pack_scatter_msg(sizes, lo: int, hi: int, frag: bytes) -> bytes:
    """_pack_scatter_msg (collectives.py:432-434)."""
    import struct

    return struct.pack("<QQQ", len(sizes), lo, hi) + np.asarray(sizes, dtype="<u8").tobytes() + frag


def scatter_counts(n: int, N: int, counts=None) -> list[int]:
    if counts is None:
        counts = [hi - lo for lo, hi in chunk_spans(n, N)]
    counts = [int(c) for c in counts]
    if len(counts) != N:
        raise ValueError(f"need {N} block counts, got {len(counts)}")
    if any(c < 0 for c in counts):
        raise ValueError("block counts must be non-negative")
    if sum(counts) != n:
        raise ValueError(f"block counts sum to {sum(counts)}, root buffer has {n} values")
    return counts


def binomial_scatter_virtual(root_data, N: int, eb, counts=None, root: int = 0, ws: Workspace | None = None,
                             trace: Trace | None = None, counters: list | None = None) -> list[torch.Tensor]:
    """binomial_scatter_c with N virtual ranks on one GPU.

    The root compresses all N blocks in ONE multi-segment launch, packed in
    virtual-rank order; the tree forwards contiguous byte ranges; each
    non-root rank decodes only its own blob; the root keeps its slice verbatim.
    """
    from .segments import compress_segments

    ebf = _check_eb(eb)
    ws = ws or Workspace()
    x = _dev_inputs([root_data], 1, ws.device)[0]
    _check_finite([x])
    counts = scatter_counts(x.numel(), N, counts)
    if not 0 <= root < N:
        raise ValueError(f"root {root} out of range [0, {N})")
    if counters is None:
        counters = [Counters() for _ in range(N)]
    lo = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    outputs = [None] * N
    outputs[root] = x[lo[root] : lo[root + 1]].clone()
    if N == 1:
        return outputs
    order = [(root + j) % N for j in range(N)]
    # gather the root's slices in virtual order (one device copy), one launch for N blobs
    xv = torch.cat([x[lo[r] : lo[r + 1]] for r in order])
    seg = compress_segments(xv, [counts[r] for r in order], ebf, ws)
    counters[root].n_compress += N
    counters[root].raw_bytes_in += 4 * x.numel()
    sizes = seg.sizes
    counters[root].blob_bytes_out += int(sum(sizes))
    if trace is not None:
        packed = seg.packed_bytes()
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        inbox = {}
        for child, clo, chi in scatter_children(0, N)[1]:
            msg = pack_scatter_msg(sizes, clo, chi, packed[offs[clo] : offs[chi - 1] + sizes[chi - 1]])
            trace.msgs.append((root, order[child], msg))
        for vr in range(1, N):
            _, sends = scatter_children(vr, N)
            for child, clo, chi in sends:
                msg = pack_scatter_msg(sizes, clo, chi, packed[offs[clo] : offs[chi - 1] + sizes[chi - 1]])
                trace.msgs.append((order[vr], order[child], msg))
        del inbox
    for vr in range(1, N):
        me = order[vr]
        outputs[me] = decompress(seg.blob(vr), ws)
        counters[me].n_decompress += 1
        if outputs[me].numel() != counts[me]:
            raise ValueError(f"rank {me} decoded {outputs[me].numel()} values, expected {counts[me]}")
    return outputs


# ---------------------------------------------------------------------------
# registry + single-process driver (collectives.py:540-574, simnet.py:225-311)
# ---------------------------------------------------------------------------

ALGORITHMS = {
    "ring-allgather": "allgather",
    "ring-reduce-scatter": "reduce_scatter",
    "ring-allreduce": "allreduce",
    "rd-allreduce": "allreduce",
    "binomial-scatter": "scatter",
    "cprp2p-allgather": "allgather",
    "lossless-allgather": "allgather",
    "lossless-reduce-scatter": "reduce_scatter",
    "lossless-allreduce": "allreduce",
    "lossless-scatter": "scatter",
}


def get_algorithm(algorithm: str) -> str:
    try:
        return ALGORITHMS[algorithm]
    except KeyError:
        raise ValueError(f"unknown algorithm {algorithm!r}; valid: {', '.join(sorted(ALGORITHMS))}") from None


@dataclass
class Report:
    algorithm: str
    ranks: int
    counters_per_rank: list
    compression_ratio: float | None
    trace: Trace | None = None


def run_collective(algorithm: str, inputs, *, ranks: int | None = None, eb: float | None = None,
                   reduce_op: str = "sum", counts=None, root: int = 0, record_payloads: bool = False,
                   workspace: Workspace | None = None):
    """Run one collective with all ranks on the current GPU (simnet.run_collective shape).

    ``inputs`` is a list of per-rank buffers, except for scatter where it is
    the root's buffer and ``ranks`` gives the communicator size.
    """
    family = get_algorithm(algorithm)
    if eb is None and not algorithm.startswith("lossless-"):
        raise ValueError("the error-bounded codec needs an error bound (eb)")
    ws = workspace or Workspace()
    trace = Trace() if record_payloads else None
    N = ranks if family == "scatter" else len(inputs)
    if N is None or N < 1:
        raise ValueError(f"communicator needs at least 1 rank, got {N}")
    counters = [Counters() for _ in range(N)]
    if algorithm == "rd-allreduce":
        out = rd_allreduce_virtual(inputs, eb, reduce_op, ws, trace, counters)
    elif algorithm == "cprp2p-allgather":
        out = cprp2p_allgather_virtual(inputs, eb, ws, trace, counters)
    elif algorithm == "lossless-allreduce":
        out = lossless_ring_allreduce(inputs, reduce_op, ws, trace, counters)
    elif algorithm == "lossless-reduce-scatter":
        out = lossless_ring_reduce_scatter(inputs, reduce_op, ws, trace, counters)
    elif algorithm == "lossless-allgather":
        out = lossless_ring_allgather(inputs, ws, trace, counters)
    elif algorithm == "lossless-scatter":
        out = lossless_binomial_scatter(inputs, N, counts, root, ws)
    elif family == "allreduce":
        out = ring_allreduce_virtual(inputs, eb, reduce_op, ws, trace, counters)
    elif family == "reduce_scatter":
        out = ring_reduce_scatter_virtual(inputs, eb, reduce_op, ws, trace, counters)
    elif family == "allgather":
        out = ring_allgather_virtual(inputs, eb, ws, trace, counters)
    else:
        out = binomial_scatter_virtual(inputs, N, eb, counts, root, ws, trace, counters)
    raw = sum(c.raw_bytes_in for c in counters)
    out_b = sum(c.blob_bytes_out for c in counters)
    cr = raw / out_b if raw > 0 and out_b > 0 else None  # simnet.py:276-278
    return out, Report(algorithm, N, [c.as_dict() for c in counters], cr, trace)
