"""Compression-enabled collectives: schedules over the device codec.

The reference (``/root/reference/pkg/src/gzccl/collectives.py``) runs every
rank in one process over a simulated network.  This module keeps its
algorithm ids, schedules, per-rank outputs, counters and message traces and
provides two drivers:

* :func:`run_collective` (``run_collective(network, algorithm, inputs, *, eb,
  reduce_op, codec, bits, counts, seed, data_source, compute_accuracy)``, the
  shape of simnet.py:225-311): all N ranks on ONE GPU in one process,
  executing the reference's two-pass step schedule with the device kernels.
  It returns the outputs and a :class:`~.metrics.CollectiveReport` with the
  lossless-rerun accuracy statistics and the compression ratio over every
  compression; ``network`` is a rank count, a :class:`CommunicatorSpec`, a
  :class:`Network` (trace + counters) or the reference's own Network object.
* :mod:`paper_2308_05199_b200.comm`: one process per GPU, blobs moved over
  NVLink peer memory (CUDA IPC) by the kernels themselves.

Key fusion (collectives.py:274-290): the chunk rank i compresses at RS step
s+1 is exactly the chunk it reduced at step s, so each RS step of the
error-bounded codec is ONE kernel ``compress(op(local, decompress(recv)))``
(csrc gz_reduce_step).  The lossless twins and the fixed-rate comparator run
the same schedules on verbatim / fixed-rate device payloads (``_generic_*``).
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .codec import BLOCK, DeviceBlob, Workspace, _check_eb, _stream, compress, decompress

REDUCE_OPS = ("sum", "max")  # collectives.py:27
_OP_CODE = {"sum": 0, "max": 1}
CODECS = ("ebz", "fixed-rate", "none")  # collectives.py:185-194


def chunk_spans(n: int, ranks: int) -> list[tuple[int, int]]:
    """Partition [0, n) into ``ranks`` chunks of ceil(n/ranks) (collectives.py:42-45)."""
    step = -(-n // ranks) if n else 0
    return [(min(c * step, n), min((c + 1) * step, n)) for c in range(ranks)]


def _check_op(op: str) -> int:
    if op not in _OP_CODE:
        raise ValueError(f"unknown reduce op {op!r}, expected one of {REDUCE_OPS}")
    return _OP_CODE[op]


# ---------------------------------------------------------------------------
# counters, traces, device timing
# ---------------------------------------------------------------------------

_OPCOUNTER_KEYS = ("n_compress", "n_decompress", "n_messages", "bytes_sent", "bytes_received", "compress_s",
                   "decompress_s", "comm_s", "reduce_s", "staging_s", "other_s")  # simnet.OpCounters, simnet.py:50-74


@dataclass
class Counters:
    """Per-rank operation counts with the fields of simnet.OpCounters.  The
    *_s phase fields hold MEASURED device seconds (CUDA events) when the run
    is timed; raw_bytes_in / blob_bytes_out are this rank's share of the
    transport totals (collectives.py:114-147)."""

    n_compress: int = 0
    n_decompress: int = 0
    n_messages: int = 0
    bytes_sent: int = 0
    bytes_received: int = 0
    compress_s: float = 0.0
    decompress_s: float = 0.0
    comm_s: float = 0.0
    reduce_s: float = 0.0
    staging_s: float = 0.0
    other_s: float = 0.0
    raw_bytes_in: int = 0
    blob_bytes_out: int = 0

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in _OPCOUNTER_KEYS}


@dataclass
class Trace:
    """Messages as (src, dst, payload bytes), like Network(record_payloads=True)."""

    msgs: list = field(default_factory=list)

    def add(self, src: int, dst: int, blob) -> None:
        self.msgs.append((src, dst, bytes(blob)))


class _Clock:
    """CUDA-event marks around every device op of a run, attributed to a rank
    and a phase (compress / decompress / reduce)."""

    def __init__(self):
        self.marks = []

    def settle(self, counters: list) -> float:
        """Add the measured seconds to the counters; return first-to-last span."""
        if not self.marks:
            return 0.0
        torch.cuda.synchronize()
        for rank, kind, e0, e1 in self.marks:
            secs = e0.elapsed_time(e1) * 1e-3
            setattr(counters[rank], kind + "_s", getattr(counters[rank], kind + "_s") + secs)
        return self.marks[0][2].elapsed_time(self.marks[-1][3]) * 1e-3


_CLOCK: _Clock | None = None


@contextlib.contextmanager
def _timed(rank: int, kind: str):
    if _CLOCK is None:
        yield
        return
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    yield
    e1.record()
    _CLOCK.marks.append((rank, kind, e0, e1))


def _deliver(counters: list, trace: Trace | None, src: int, dst: int, nbytes: int, payload=None) -> None:
    """Account one message src -> dst (simnet.py:119-137): sender n_messages /
    bytes_sent, receiver bytes_received; payload() is only built when traced."""
    counters[src].n_messages += 1
    counters[src].bytes_sent += nbytes
    counters[dst].bytes_received += nbytes
    if trace is not None:
        trace.add(src, dst, payload() if callable(payload) else payload)


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------


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


def apply_op(op: str, local: torch.Tensor, received: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """_apply_op (collectives.py:32-39) on the device: local + received, or
    np.maximum(local, received); one kernel (gz_apply_op)."""
    opc = _check_op(op)
    if local.numel() != received.numel():
        raise ValueError(f"reduce shape mismatch: ({local.numel()},) vs ({received.numel()},)")
    out = torch.empty_like(local) if out is None else out
    L.check(L.lib().gz_apply_op(local.data_ptr(), received.data_ptr(), out.data_ptr(), local.numel(), opc,
                                _stream()), "gz_apply_op")
    return out


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


def _check_finite(bufs, ws: Workspace | None = None) -> None:
    """codec._ingest's finiteness scan (codec.py:79-86) of every buffer, in
    rank order, on the device (gz_copy_checked without a destination)."""
    lib = L.lib()
    for b in bufs:
        if b.numel() == 0:
            continue
        w = ws or Workspace(b.device)
        w.reset_status()
        L.check(lib.gz_copy_checked(b.data_ptr(), None, b.numel(), 0, w.status_ptr(), _stream()), "gz_copy_checked")
        st = w.read_status()
        if st[0] != (1 << 64) - 1:
            raise ValueError(f"non-finite value at offset {int(st[0])}")


def _new_counters(N: int, counters):
    return [Counters() for _ in range(N)] if counters is None else counters


# ---------------------------------------------------------------------------
# error-bounded codec: fused device schedules
# ---------------------------------------------------------------------------


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
    _check_finite(bufs, ws)
    counters = _new_counters(N, counters)
    if N == 1:
        return ([bufs[0].clone()], [None]) if _keep_blobs else [bufs[0].clone()]
    spans = chunk_spans(n, N)

    def chunk(i, c):
        lo, hi = spans[c]
        return bufs[i][lo:hi]

    # step 0 sends: rank i compresses its own chunk i
    sending = []
    for i in range(N):
        with _timed(i, "compress"):
            blob = compress(chunk(i, i), ebf, ws)
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * blob.n
        counters[i].blob_bytes_out += len(blob)
        sending.append(blob)
    owned = [None] * N
    for s in range(N - 1):
        for i in range(N):
            _deliver(counters, trace, i, (i + 1) % N, len(sending[i]), sending[i].tobytes)
        nxt = []
        for i in range(N):
            recv = sending[(i - 1) % N]
            c_in = (i - s - 1) % N
            last = s == N - 2
            acc = torch.empty(spans[c_in][1] - spans[c_in][0], dtype=torch.float32, device=ws.device) if last else None
            with _timed(i, "reduce"):  # decode + op + re-encode, one kernel
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
        for i in range(N):
            _deliver(counters, trace, i, (i + 1) % N, len(carry[i]), carry[i].tobytes)
        carry = [carry[(i - 1) % N] for i in range(N)]
        for i in range(N):
            with _timed(i, "decompress"):
                gathered[i][chunk_of((i - 1 - s) % N)] = decompress(carry[i], ws)
            counters[i].n_decompress += 1
    return gathered


def ring_allreduce_virtual(buffers, eb, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                           counters: list | None = None) -> list[torch.Tensor]:
    """ring_allreduce_c (collectives.py:294-308): RS, then compress-once AG."""
    ws = ws or Workspace()
    N = len(buffers)
    counters = _new_counters(N, counters)
    if N == 1:
        bufs = _dev_inputs(buffers, 1, ws.device)
        _check_finite(bufs, ws)
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
    _check_finite(owned, ws)
    counters = _new_counters(N, counters)
    if N == 1:
        return [owned[0].clone()]
    blobs = []
    for i in range(N):
        with _timed(i, "compress"):
            blobs.append(compress(owned[i], ebf, ws))
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * owned[i].numel()
        counters[i].blob_bytes_out += len(blobs[-1])
    gathered = _allgather_blobs(blobs, owned, lambda i: i, ws, trace, counters)
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


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
    _check_finite(data, ws)
    data = [d.clone() for d in data]
    counters = _new_counters(N, counters)
    if N == 1:
        return data
    pof2, r, steps, role, remapped, actual = rd_plan(N)
    donors = [i for i in range(N) if role(i) == "donor"]
    parts = [i for i in range(N) if role(i) != "donor"]

    def send(i, dst, blob):
        _deliver(counters, trace, i, dst, len(blob), blob.tobytes)

    def comp(i):
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * data[i].numel()
        with _timed(i, "compress"):
            b = compress(data[i], ebf, ws)
        counters[i].blob_bytes_out += len(b)
        return b

    def fused(i, recv):  # data[i] = op(data[i], dec(recv)); returns compress(data[i])
        counters[i].n_decompress += 1
        counters[i].n_compress += 1
        counters[i].raw_bytes_in += 4 * data[i].numel()
        with _timed(i, "reduce"):
            b = reduce_step(recv, data[i], ebf, op, ws, acc_out=data[i])
        counters[i].blob_bytes_out += len(b)
        return b

    def last(i, recv):  # data[i] = op(data[i], dec(recv))
        counters[i].n_decompress += 1
        with _timed(i, "reduce"):
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
            with _timed(i, "decompress"):
                data[i] = decompress(nxt[i + 1], ws)
    return data


def cprp2p_allgather_virtual(chunks, eb, ws: Workspace | None = None, trace: Trace | None = None,
                             counters: list | None = None) -> list[torch.Tensor]:
    """cprp2p_allgather (collectives.py:311-341): the compress-per-hop baseline;
    every hop decompresses and re-compresses, so a chunk that travelled h hops
    carries up to h * eb of error (N-1 compressions and decompressions per rank)."""
    ebf = _check_eb(eb)
    ws = ws or Workspace()
    N = len(chunks)
    owned = _dev_inputs(chunks, N, ws.device)
    _check_finite(owned, ws)
    counters = _new_counters(N, counters)
    if N == 1:
        return [owned[0].clone()]
    gathered = [{i: owned[i]} for i in range(N)]
    current = list(owned)
    for s in range(N - 1):
        sent = []
        for i in range(N):
            with _timed(i, "compress"):
                b = compress(current[i], ebf, ws)
            counters[i].n_compress += 1
            counters[i].raw_bytes_in += 4 * current[i].numel()
            counters[i].blob_bytes_out += len(b)
            sent.append(b)
            _deliver(counters, trace, i, (i + 1) % N, len(b), b.tobytes)
        for i in range(N):
            with _timed(i, "decompress"):
                vals = decompress(sent[(i - 1) % N], ws)
            counters[i].n_decompress += 1
            gathered[i][(i - 1 - s) % N] = vals
            current[i] = vals
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


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


def _scatter_trace(trace: Trace | None, counters: list, root: int, order: list, sizes: list, packed: callable):
    """Account / record the tree's messages (collectives.py:500-525): each one
    carries the size table and a contiguous byte range of the packed blobs."""
    N = len(order)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    payload = packed() if trace is not None else None

    def emit(src, child, clo, chi):
        nbytes = scatter_msg_overhead(N) + int(offs[chi] - offs[clo])
        msg = None
        if payload is not None:
            msg = pack_scatter_msg(sizes, clo, chi, payload[offs[clo]: offs[chi - 1] + sizes[chi - 1]])
        _deliver(counters, trace, src, order[child], nbytes, msg)

    for child, clo, chi in scatter_children(0, N)[1]:
        emit(root, child, clo, chi)
    for vr in range(1, N):
        for child, clo, chi in scatter_children(vr, N)[1]:
            emit(order[vr], child, clo, chi)


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
    _check_finite([x], ws)
    counts = scatter_counts(x.numel(), N, counts)
    if not 0 <= root < N:
        raise ValueError(f"root {root} out of range [0, {N})")
    counters = _new_counters(N, counters)
    lo = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    outputs = [None] * N
    outputs[root] = x[lo[root] : lo[root + 1]].clone()
    if N == 1:
        return outputs
    order = [(root + j) % N for j in range(N)]
    # gather the root's slices in virtual order (one device copy), one launch for N blobs
    xv = torch.cat([x[lo[r] : lo[r + 1]] for r in order])
    with _timed(root, "compress"):
        seg = compress_segments(xv, [counts[r] for r in order], ebf, ws)
    counters[root].n_compress += N
    counters[root].raw_bytes_in += 4 * x.numel()
    sizes = seg.sizes
    counters[root].blob_bytes_out += int(sum(sizes))
    _scatter_trace(trace, counters, root, order, sizes, seg.packed_bytes)
    for vr in range(1, N):
        me = order[vr]
        with _timed(me, "decompress"):
            outputs[me] = decompress(seg.blob(vr), ws)
        counters[me].n_decompress += 1
        if outputs[me].numel() != counts[me]:
            raise ValueError(f"rank {me} decoded {outputs[me].numel()} values, expected {counts[me]}")
    return outputs


# ---------------------------------------------------------------------------
# verbatim / fixed-rate payloads: the same schedules, unfused (collectives.py:94-194)
# ---------------------------------------------------------------------------


class _RawDev:
    """RawTransport (collectives.py:94-111) on the device: verbatim float32
    payloads, no kernels, no counters, no loss."""

    name = "none"

    def __init__(self, counters: list, ws: Workspace):
        self.counters = counters

    def enc(self, i: int, t: torch.Tensor) -> torch.Tensor:
        return t.clone()

    def dec(self, i: int, m: torch.Tensor) -> torch.Tensor:
        return m.clone()

    def enc_blocks(self, i: int, blocks: list) -> list:
        return [b.clone() for b in blocks]

    @staticmethod
    def size(m) -> int:
        return 4 * m.numel()

    @staticmethod
    def payload(m) -> bytes:
        return m.cpu().numpy().astype("<f4").tobytes()


class _FixedRateDev:
    """FixedRateTransport (collectives.py:150-182) on the device (gz_fr_*)."""

    name = "fixed-rate"

    def __init__(self, counters: list, ws: Workspace, bits: int):
        self.counters, self.ws, self.bits = counters, ws, int(bits)

    def enc(self, i: int, t: torch.Tensor) -> torch.Tensor:
        from .codec import fixed_rate_compress

        with _timed(i, "compress"):
            m = fixed_rate_compress(t, self.bits, self.ws)
        c = self.counters[i]
        c.n_compress += 1
        c.raw_bytes_in += 4 * t.numel()
        c.blob_bytes_out += m.numel()
        return m

    def dec(self, i: int, m: torch.Tensor) -> torch.Tensor:
        from .codec import fixed_rate_decompress

        with _timed(i, "decompress"):
            v = fixed_rate_decompress(m, self.ws)
        self.counters[i].n_decompress += 1
        return v

    def enc_blocks(self, i: int, blocks: list) -> list:
        return [self.enc(i, b) for b in blocks]

    @staticmethod
    def size(m) -> int:
        return m.numel()

    @staticmethod
    def payload(m) -> bytes:
        return m.cpu().numpy().tobytes()


def _dev_op(i: int, op: str, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    with _timed(i, "reduce"):
        return apply_op(op, a, b)


def _generic_reduce_scatter(bufs, op, tr, trace, counters):
    """ring_reduce_scatter_c (collectives.py:258-291) over a device transport."""
    N = len(bufs)
    n = _require_equal(bufs)
    if N == 1:
        return [bufs[0].clone()]
    spans = chunk_spans(n, N)
    acc = [[b[lo:hi].clone() for lo, hi in spans] for b in bufs]
    for s in range(N - 1):
        sent = [tr.enc(i, acc[i][(i - s) % N]) for i in range(N)]
        for i in range(N):
            _deliver(counters, trace, i, (i + 1) % N, tr.size(sent[i]), lambda m=sent[i]: tr.payload(m))
        for i in range(N):
            vals = tr.dec(i, sent[(i - 1) % N])
            c_in = (i - s - 1) % N
            acc[i][c_in] = _dev_op(i, op, acc[i][c_in], vals)
    return [acc[i][(i + 1) % N] for i in range(N)]


def _generic_allgather(owned, chunk_of, tr, trace, counters):
    """_ring_allgather (collectives.py:215-244): encode once at the owner, forward the bytes."""
    N = len(owned)
    gathered = [{chunk_of(i): owned[i]} for i in range(N)]
    if N == 1:
        return gathered
    carry = [None] * N
    for s in range(N - 1):
        for i in range(N):
            if s == 0:
                carry[i] = tr.enc(i, owned[i])
            _deliver(counters, trace, i, (i + 1) % N, tr.size(carry[i]), lambda m=carry[i]: tr.payload(m))
        carry = [carry[(i - 1) % N] for i in range(N)]
        for i in range(N):
            gathered[i][chunk_of((i - 1 - s) % N)] = tr.dec(i, carry[i])
    return gathered


def _generic_cprp2p(owned, tr, trace, counters):
    """cprp2p_allgather (collectives.py:311-341) over a device transport."""
    N = len(owned)
    if N == 1:
        return [owned[0].clone()]
    gathered = [{i: owned[i]} for i in range(N)]
    current = list(owned)
    for s in range(N - 1):
        sent = [tr.enc(i, current[i]) for i in range(N)]
        for i in range(N):
            _deliver(counters, trace, i, (i + 1) % N, tr.size(sent[i]), lambda m=sent[i]: tr.payload(m))
        for i in range(N):
            vals = tr.dec(i, sent[(i - 1) % N])
            gathered[i][(i - 1 - s) % N] = vals
            current[i] = vals
    return [torch.cat([gathered[i][c] for c in range(N)]) for i in range(N)]


def _generic_rd(bufs, op, tr, trace, counters):
    """rd_allreduce_c (collectives.py:349-424) over a device transport."""
    N = len(bufs)
    _require_equal(bufs)
    data = [b.clone() for b in bufs]
    if N == 1:
        return data
    pof2, r, steps, role, remapped, actual = rd_plan(N)
    donors = [i for i in range(N) if role(i) == "donor"]
    parts = [i for i in range(N) if role(i) != "donor"]

    def post(i, dst, m):
        _deliver(counters, trace, i, dst, tr.size(m), lambda: tr.payload(m))

    if r:
        msgs = {i: tr.enc(i, data[i]) for i in donors}
        for i in donors:
            post(i, i + 1, msgs[i])
        for i in donors:
            data[i + 1] = _dev_op(i + 1, op, data[i + 1], tr.dec(i + 1, msgs[i]))
    for t in range(steps):
        partner = {i: actual(remapped(i) ^ (1 << t)) for i in parts}
        msgs = {i: tr.enc(i, data[i]) for i in parts}
        for i in parts:
            post(i, partner[i], msgs[i])
        for i in parts:
            data[i] = _dev_op(i, op, data[i], tr.dec(i, msgs[partner[i]]))
    if r:
        msgs = {i + 1: tr.enc(i + 1, data[i + 1]) for i in donors}
        for i in donors:
            post(i + 1, i, msgs[i + 1])
        for i in donors:
            data[i] = tr.dec(i, msgs[i + 1])
    return data


def _generic_scatter(x, N, counts, root, tr, trace, counters):
    """binomial_scatter_c (collectives.py:467-532) over a device transport."""
    lo = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    outputs = [None] * N
    outputs[root] = x[lo[root]: lo[root + 1]].clone()
    if N == 1:
        return outputs
    order = [(root + j) % N for j in range(N)]
    msgs = tr.enc_blocks(root, [x[lo[r]: lo[r + 1]] for r in order])
    sizes = [tr.size(m) for m in msgs]
    _scatter_trace(trace, counters, root, order, sizes, lambda: b"".join(tr.payload(m) for m in msgs))
    for vr in range(1, N):
        me = order[vr]
        outputs[me] = tr.dec(me, msgs[vr])
        if outputs[me].numel() != counts[me]:
            raise ValueError(f"rank {me} decoded {outputs[me].numel()} values, expected {counts[me]}")
    return outputs


# lossless twins (collectives.py:560-566): the schedules with verbatim payloads

def lossless_ring_reduce_scatter(buffers, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                                 counters: list | None = None):
    _check_op(op)
    ws = ws or Workspace()
    bufs = _dev_inputs(buffers, len(buffers), ws.device)
    _check_finite(bufs, ws)
    counters = _new_counters(len(bufs), counters)
    return _generic_reduce_scatter(bufs, op, _RawDev(counters, ws), trace, counters)


def lossless_ring_allgather(chunks, ws: Workspace | None = None, trace: Trace | None = None,
                            counters: list | None = None):
    ws = ws or Workspace()
    N = len(chunks)
    owned = _dev_inputs(chunks, N, ws.device)
    _check_finite(owned, ws)
    counters = _new_counters(N, counters)
    g = _generic_allgather(owned, lambda i: i, _RawDev(counters, ws), trace, counters)
    return [torch.cat([g[i][c] for c in range(N)]) if N > 1 else owned[0].clone() for i in range(N)]


def lossless_ring_allreduce(buffers, op="sum", ws: Workspace | None = None, trace: Trace | None = None,
                            counters: list | None = None):
    _check_op(op)
    ws = ws or Workspace()
    N = len(buffers)
    bufs = _dev_inputs(buffers, N, ws.device)
    _check_finite(bufs, ws)
    counters = _new_counters(N, counters)
    tr = _RawDev(counters, ws)
    owned = _generic_reduce_scatter(bufs, op, tr, trace, counters)
    if N == 1:
        return owned
    g = _generic_allgather(owned, lambda i: (i + 1) % N, tr, trace, counters)
    return [torch.cat([g[i][c] for c in range(N)]) for i in range(N)]


def lossless_binomial_scatter(root_data, N: int, counts=None, root: int = 0, ws: Workspace | None = None,
                              trace: Trace | None = None, counters: list | None = None):
    """binomial_scatter_c with the RawTransport: every rank gets its slice verbatim."""
    ws = ws or Workspace()
    x = _dev_inputs([root_data], 1, ws.device)[0]
    _check_finite([x], ws)
    counts = scatter_counts(x.numel(), N, counts)
    counters = _new_counters(N, counters)
    return _generic_scatter(x, N, counts, root, _RawDev(counters, ws), trace, counters)


# ---------------------------------------------------------------------------
# registry + single-process driver (collectives.py:540-574, simnet.py:225-311)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class AlgoInfo:
    """Algorithm id, family and whether it is a lossless twin (collectives.py:540-553)."""

    id: str
    family: str  # allgather | reduce_scatter | allreduce | scatter
    lossless: bool = False


ALGORITHMS = {a.id: a for a in [
    AlgoInfo("ring-allgather", "allgather"),
    AlgoInfo("ring-reduce-scatter", "reduce_scatter"),
    AlgoInfo("ring-allreduce", "allreduce"),
    AlgoInfo("rd-allreduce", "allreduce"),
    AlgoInfo("binomial-scatter", "scatter"),
    AlgoInfo("cprp2p-allgather", "allgather"),
    AlgoInfo("lossless-allgather", "allgather", True),
    AlgoInfo("lossless-reduce-scatter", "reduce_scatter", True),
    AlgoInfo("lossless-allreduce", "allreduce", True),
    AlgoInfo("lossless-scatter", "scatter", True),
]}


def get_algorithm(algorithm: str) -> AlgoInfo:
    try:
        return ALGORITHMS[algorithm]
    except KeyError:
        raise ValueError(f"unknown algorithm {algorithm!r}; valid: {', '.join(sorted(ALGORITHMS))}") from None


@dataclass
class CommunicatorSpec:
    """Rank count and the root of rooted collectives (simnet.py:36-47)."""

    size: int
    root: int = 0

    def __post_init__(self):
        if self.size < 1:
            raise ValueError(f"communicator needs at least 1 rank, got {self.size}")
        if not 0 <= self.root < self.size:
            raise ValueError(f"root {self.root} out of range [0, {self.size})")


@dataclass
class _RankView:
    id: int
    counters: Counters = field(default_factory=Counters)


class Network:
    """What a caller of the reference's run_collective reads back from its
    network besides the report: per-rank counters and, with
    ``record_payloads``, the message trace [(src, dst, len, payload)]
    (simnet.py:77-117).  There is no simulated clock: the collectives run on
    the device and their seconds are measured."""

    def __init__(self, spec: CommunicatorSpec, params=None, record_payloads: bool = False):
        self.spec = spec
        self.params = params
        self.record_payloads = record_payloads
        self.ranks = [_RankView(i) for i in range(spec.size)]
        self.trace: list = []

    @property
    def size(self) -> int:
        return self.spec.size

    @property
    def root(self) -> int:
        return self.spec.root


def create_network(spec: CommunicatorSpec, params=None, **kw) -> Network:
    return Network(spec, params, **kw)


def _spec_of(network) -> tuple[int, int]:
    if isinstance(network, int):
        return CommunicatorSpec(network).size, 0
    spec = getattr(network, "spec", network)
    return int(spec.size), int(getattr(spec, "root", 0))


def _run_algo(info: AlgoInfo, codec: str, N: int, root: int, inputs, eb, bits, reduce_op, counts, ws, trace,
              counters):
    """Dispatch one algorithm: the fused error-bounded schedules for codec
    "ebz", the generic device transports otherwise."""
    fam = info.family
    if codec == "ebz":
        if info.id == "rd-allreduce":
            return rd_allreduce_virtual(inputs, eb, reduce_op, ws, trace, counters)
        if info.id == "cprp2p-allgather":
            return cprp2p_allgather_virtual(inputs, eb, ws, trace, counters)
        if fam == "allreduce":
            return ring_allreduce_virtual(inputs, eb, reduce_op, ws, trace, counters)
        if fam == "reduce_scatter":
            return ring_reduce_scatter_virtual(inputs, eb, reduce_op, ws, trace, counters)
        if fam == "allgather":
            return ring_allgather_virtual(inputs, eb, ws, trace, counters)
        return binomial_scatter_virtual(inputs, N, eb, counts, root, ws, trace, counters)
    tr = _RawDev(counters, ws) if codec == "none" else _FixedRateDev(counters, ws, bits)
    if fam == "scatter":
        x = _dev_inputs([inputs], 1, ws.device)[0]
        _check_finite([x], ws)
        if not 0 <= root < N:
            raise ValueError(f"root {root} out of range [0, {N})")
        return _generic_scatter(x, N, scatter_counts(x.numel(), N, counts), root, tr, trace, counters)
    bufs = _dev_inputs(inputs, N, ws.device)
    _check_finite(bufs, ws)
    if fam in ("allreduce", "reduce_scatter"):
        _check_op(reduce_op)
        _require_equal(bufs)
    if info.id == "rd-allreduce":
        return _generic_rd(bufs, reduce_op, tr, trace, counters)
    if info.id == "cprp2p-allgather":
        return _generic_cprp2p(bufs, tr, trace, counters)
    if fam == "allgather":
        g = _generic_allgather(bufs, lambda i: i, tr, trace, counters)
        return [torch.cat([g[i][c] for c in range(N)]) if N > 1 else bufs[0].clone() for i in range(N)]
    owned = _generic_reduce_scatter(bufs, reduce_op, tr, trace, counters)
    if fam == "reduce_scatter" or N == 1:
        return owned
    g = _generic_allgather(owned, lambda i: (i + 1) % N, tr, trace, counters)
    return [torch.cat([g[i][c] for c in range(N)]) for i in range(N)]


def run_collective(network, algorithm: str, inputs, *, eb: float | None = None, reduce_op: str = "sum",
                   codec: str = "ebz", bits: int = 8, counts=None, seed: int | None = None,
                   data_source: str | None = None, compute_accuracy: bool = True,
                   record_payloads: bool | None = None, workspace: Workspace | None = None):
    """Run one collective with all ranks on the current GPU (simnet.run_collective, simnet.py:225-311).

    ``network``: a rank count, a :class:`CommunicatorSpec`, a :class:`Network`
    or the reference's Network / CommunicatorSpec (its size and root are used;
    a network's per-rank counters and, with record_payloads, its trace are
    filled like simnet's).  ``inputs``: per-rank buffers, except for the
    scatter family (the root's full buffer).  numpy / array-like inputs give
    numpy outputs, CUDA tensors give CUDA tensors.  The report carries the
    aggregated counters, measured device seconds, the accuracy against the
    same schedule rerun with verbatim payloads (so only codec distortion
    remains) and the compression ratio over every compression of the run.
    """
    global _CLOCK
    from .metrics import AccuracyStats, CollectiveReport

    info = get_algorithm(algorithm)
    if info.lossless:
        codec = "none"
    if codec not in CODECS:
        raise ValueError(f"unknown codec {codec!r}, expected 'ebz', 'fixed-rate', or 'none'")
    if codec == "ebz":
        if eb is None:
            raise ValueError("the error-bounded codec needs an error bound (eb)")
        eb = _check_eb(eb)
    N, root = _spec_of(network)
    if N < 1:
        raise ValueError(f"communicator needs at least 1 rank, got {N}")
    ws = workspace or Workspace()
    if record_payloads is None:
        record_payloads = bool(getattr(network, "record_payloads", False))
    trace = Trace() if record_payloads else None
    counters = [Counters() for _ in range(N)]
    as_numpy = not (isinstance(inputs, torch.Tensor) or (isinstance(inputs, (list, tuple)) and inputs
                                                          and isinstance(inputs[0], torch.Tensor)))
    clock = _Clock()
    _CLOCK = clock
    try:
        outputs = _run_algo(info, codec, N, root, inputs, eb, bits, reduce_op, counts, ws, trace, counters)
    finally:
        _CLOCK = None
    makespan = clock.settle(counters)

    lossless_run = info.lossless or codec == "none"
    flat_out = torch.cat([o.reshape(-1) for o in outputs]) if outputs else torch.empty(0, device=ws.device)
    if compute_accuracy and not lossless_run:
        # the lossless oracle: the same schedule with verbatim payloads, so the
        # reduction order matches and only codec distortion remains (simnet.py:257-264)
        ref = _run_algo(info, "none", N, root, inputs, eb, bits, reduce_op, counts, ws, None,
                        [Counters() for _ in range(N)])
        accuracy = AccuracyStats.of(torch.cat([o.reshape(-1) for o in ref]), flat_out)
    else:
        accuracy = AccuracyStats.of(flat_out, flat_out)

    raw_in = sum(c.raw_bytes_in for c in counters)
    blob_out = sum(c.blob_bytes_out for c in counters)
    cr = raw_in / blob_out if raw_in > 0 and blob_out > 0 else None  # simnet.py:276-278
    total = {k: sum(getattr(c, k) for c in counters) for k in _OPCOUNTER_KEYS}
    phase = {k: total[k + "_s"] for k in ("compress", "decompress", "comm", "reduce", "staging", "other")}
    if info.family == "scatter":
        elements_per_rank, total_elements = None, int(_numel(inputs))
    else:
        elements_per_rank = int(_numel(inputs[0])) if len(inputs) else 0
        total_elements = int(sum(_numel(b) for b in inputs))
    report = CollectiveReport(
        algorithm=algorithm, ranks=N, root=root, elements_per_rank=elements_per_rank,
        total_elements=total_elements, eb=float(eb) if eb is not None and not lossless_run and codec == "ebz" else None,
        codec="none" if info.lossless else codec,
        reduce_op=reduce_op if info.family in ("reduce_scatter", "allreduce") else None,
        counters=total, counters_per_rank=[c.as_dict() for c in counters], phase_seconds=phase,
        makespan_seconds=makespan, accuracy=accuracy, compression_ratio=cr,
        flags={"overlap": True, "staging": False, "multi_stream": True}, seed=seed, data_source=data_source,
        extra={"device": str(ws.device), "timing": "measured device seconds, all ranks on one GPU"})
    _fill_network(network, counters, trace)
    if as_numpy:
        outputs = [o.cpu().numpy() for o in outputs]
    return outputs, report


def _numel(b) -> int:
    return b.numel() if isinstance(b, torch.Tensor) else int(np.asarray(b).size)


def _fill_network(network, counters: list, trace: Trace | None) -> None:
    """Mirror simnet's side effects on a network object, when one was given."""
    ranks = getattr(network, "ranks", None)
    if ranks is not None:
        for rv, c in zip(ranks, counters):
            rc = getattr(rv, "counters", None)
            if rc is None:
                continue
            for k in _OPCOUNTER_KEYS:
                if hasattr(rc, k):
                    setattr(rc, k, getattr(rc, k) + getattr(c, k))
    tr = getattr(network, "trace", None)
    if tr is not None and trace is not None:
        for s, d, b in trace.msgs:
            tr.append((s, d, len(b), b))
