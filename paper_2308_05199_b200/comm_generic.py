"""The comparator collectives on the real one-process-per-GPU path
(collectives.py:94-194, 311-341, 553-566): the lossless twins (verbatim f32
messages), the fixed-rate transport, and the compress-per-hop allgather, run
with the reference's ring schedules over NVLink peer memory.

Unlike the error-bounded ring of :mod:`comm` (fused decode + op + encode
steps, slotted messages), these move each message through a slot in the
sender's memory: the sender encodes (verbatim copy, gz_fr_compress, or
gz_compress for the per-hop allgather) into its slot and posts the receiver's
flag; the receiver pulls the slot over NVLink and decodes it (or, verbatim,
reduces straight out of the peer's memory with gz_apply_op) and posts the
sender's "consumed" flag.  Flags carry the call's epoch, so consecutive calls
never overwrite a slot a peer is still reading.  Every output is the
reference schedule's, bit for bit (tests/mgpu_worker.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .codec import _check_eb
from .collectives import _check_op, chunk_spans
from .comm import Communicator, _al, _open_peers

class _GenLayout:
    """Flags (ready[N] / consumed[N] per message slot, ready/consumed[N] for the
    allgather's owned message), then N-1 ring slots + the owned slot."""

    def __init__(self, world: int, slot_bytes: int):
        self.world = world
        self.nslots = world  # world-1 ring slots + the owned (allgather) slot
        off = _al(4 * 4 * self.nslots * world)
        self.slot_bytes = _al(slot_bytes)
        self.slot = []
        for _ in range(self.nslots):
            self.slot.append(off)
            off += self.slot_bytes
        self.total = off

    def ready(self, k, src):  # message k from rank src has landed (in the RECEIVER's flags)
        return 4 * (k * self.world + src)

    def consumed(self, k, dst):  # rank dst has read our message k (in the SENDER's flags)
        return 4 * (self.nslots * self.world + k * self.world + dst)


def _msg_bytes(codec: str, m: int, bits: int) -> int:
    lib = L.lib()
    if codec == "none":
        return 4 * m
    if codec == "fixed-rate":
        return int(lib.gz_fr_bound(m, bits))
    return _al(int(lib.gz_compress_bound(m))) + int(lib.gz_sidecar_bytes(m)) + 64  # blob, then its sidecar


def _setup(self, codec: str, m: int, bits: int):
    key = (codec, m, bits)
    if getattr(self, "_gen_key", None) == key:
        return
    _gen_close(self)
    self._gen_layout = _GenLayout(self.world, _msg_bytes(codec, m, bits))
    self._gen_buf = torch.zeros(self._gen_layout.total, dtype=torch.uint8, device=self.device)
    torch.cuda.synchronize(self.device)
    self._gen_peer = _open_peers(self, self._gen_buf)
    self._gen_key = key
    self._gen_epoch = 0
    self._gen_last = {}
    self._gen_tmp = torch.empty(max(m, 1), dtype=torch.float32, device=self.device)
    dist.barrier(group=self.group)


def _gen_close(self):
    peers = getattr(self, "_gen_peer", None)
    if peers is not None:
        lib = L.lib()
        torch.cuda.synchronize(self.device)
        for r, p in enumerate(peers):
            if r != self.rank and p:
                lib.gz_ipc_close(p)
    self._gen_peer = None
    self._gen_buf = None
    self._gen_key = None


class _Ring:
    """One call's message plumbing: encode into a slot, post, pull + decode."""

    def __init__(self, comm: Communicator, codec: str, eb, bits: int, op: str):
        self.c = comm
        self.codec, self.eb, self.bits, self.op = codec, eb, bits, op
        self.lib = L.lib()
        self.s = torch.cuda.current_stream(comm.device).cuda_stream
        self.lay = comm._gen_layout
        self.peer = comm._gen_peer
        self.prev = comm._gen_epoch
        self.e = comm._gen_epoch + 1
        self.launches = 0

    def at(self, r: int, off: int) -> int:
        return self.peer[r] + off

    def wait(self, off: int, v: int):
        if v > 0:
            L.check(self.lib.gz_stream_wait_u32_geq(self.s, self.at(self.c.rank, off), v), "gz_stream_wait_u32_geq")

    def post(self, r: int, off: int):
        L.check(self.lib.gz_stream_write_u32(self.s, self.at(r, off), self.e), "gz_stream_write_u32")

    def send(self, k: int, t: torch.Tensor, dsts):
        """encode t into our slot k (after every reader of its previous contents
        is done), then post message k to dsts"""
        me = self.c.rank
        last = self.c._gen_last  # (slot, reader) -> epoch of the last call that sent it that slot
        for d in dsts:
            self.wait(self.lay.consumed(k, d), last.get((k, d), 0))
            last[(k, d)] = self.e
        slot = self.at(me, self.lay.slot[k])
        n = t.numel()
        if self.codec == "none":
            if n:
                L.check(self.lib.gz_copy_checked(t.data_ptr(), slot, n, 0, self.c.ws.status_ptr(), self.s),
                        "gz_copy_checked")
        elif self.codec == "fixed-rate":
            scratch = self.c.ws.get("gen.fr", int(self.lib.gz_fr_workspace_bytes()))
            L.check(self.lib.gz_fr_compress(t.data_ptr(), n, self.bits, slot, self.lay.slot_bytes,
                                            self.c.ws.len_ptr(), scratch.data_ptr(), self.c.ws.status_ptr(), self.s),
                    "gz_fr_compress")
        else:  # error-bounded blob + its sidecar (the compress-per-hop allgather)
            cap = int(self.lib.gz_compress_bound(n))
            tws = self.c.ws.tile_ws(int(self.lib.gz_workspace_bytes(n)))
            L.check(self.lib.gz_compress(t.data_ptr(), n, self.eb, 32, slot, cap, self.c.ws.len_ptr(),
                                         slot + _al(cap), None, tws.data_ptr(), tws.numel(), self.c.ws.status_ptr(),
                                         self.s), "gz_compress")
        self.launches += 1
        for d in dsts:
            self.post(d, self.lay.ready(k, me))

    def recv(self, k: int, src: int, out: torch.Tensor, reduce: bool):
        """pull message k of src over NVLink: out = decode(msg), or op(out, decode(msg))"""
        self.wait(self.lay.ready(k, src), self.e)
        n = out.numel()
        slot = self.at(src, self.lay.slot[k])
        if n:
            opc = _check_op(self.op)
            if self.codec == "none":
                if reduce:
                    L.check(self.lib.gz_apply_op(out.data_ptr(), slot, out.data_ptr(), n, opc, self.s), "gz_apply_op")
                else:
                    L.check(self.lib.gz_copy_checked(slot, out.data_ptr(), n, 0, self.c.ws.status_ptr(), self.s),
                            "gz_copy_checked")
            else:
                dst = self.c._gen_tmp[:n] if reduce else out
                if self.codec == "fixed-rate":
                    L.check(self.lib.gz_fr_decompress(slot, n, self.bits, dst.data_ptr(), self.s), "gz_fr_decompress")
                else:
                    cap = int(self.lib.gz_compress_bound(n))
                    L.check(self.lib.gz_decompress_sidecar(slot, slot + _al(cap), n, self.eb, dst.data_ptr(),
                                                           self.c.ws.status_ptr(), self.s), "gz_decompress_sidecar")
                if reduce:
                    L.check(self.lib.gz_apply_op(out.data_ptr(), dst.data_ptr(), out.data_ptr(), n, opc, self.s),
                            "gz_apply_op")
            self.launches += 1
        self.post(src, self.lay.consumed(k, self.c.rank))

    def done(self):
        self.c._gen_epoch = self.e
        self.c.launches_per_call = self.launches


def _prepare(self, x, codec, eb, bits, op):
    if codec not in ("none", "fixed-rate", "ebz"):
        raise ValueError(f"unknown codec {codec!r}, expected 'ebz', 'fixed-rate', or 'none'")
    if codec == "fixed-rate" and not 1 <= int(bits) <= 16:
        raise ValueError(f"bits_per_value must be in [1, 16], got {bits}")
    x = self._check_input(x)
    _check_op(op)
    return x, (_check_eb(eb) if codec == "ebz" else None), int(bits)


def _reduce_scatter_into(ring: _Ring, work: torch.Tensor, spans):
    """ring_reduce_scatter_c (collectives.py:258-291): slot s carries our chunk (i - s)."""
    N, i = ring.c.world, ring.c.rank
    right, left = (i + 1) % N, (i - 1) % N
    for s in range(N - 1):
        lo, hi = spans[(i - s) % N]
        ring.send(s, work[lo:hi], [right])
        lo, hi = spans[(i - s - 1) % N]
        ring.recv(s, left, work[lo:hi], reduce=True)


def _allgather_owned(ring: _Ring, out: torch.Tensor, spans, chunk_of):
    """_ring_allgather (collectives.py:215-244) with a direct pull: every owner's
    message is encoded ONCE and read by all peers (the ring forwards the same bytes)."""
    N, i = ring.c.world, ring.c.rank
    k = N - 1  # the owned slot
    lo, hi = spans[chunk_of(i)]
    ring.send(k, out[lo:hi], [j for j in range(N) if j != i])
    for step in range(N - 1):
        j = (i - 1 - step) % N  # arrival order of the reference ring
        lo, hi = spans[chunk_of(j)]
        ring.recv(k, j, out[lo:hi], reduce=False)


def generic_allreduce(self, x: torch.Tensor, codec: str = "none", eb: float | None = None, bits: int = 8,
                      op: str = "sum", out: torch.Tensor | None = None, check: bool = True):
    """ring_allreduce_c with RawTransport ("none", the lossless-allreduce twin) or
    FixedRateTransport ("fixed-rate"), collectives.py:294-308 / 94-182: verbatim or
    fixed-rate messages, every reduction op(local, received) in the reference order."""
    x, ebf, bits = _prepare(self, x, codec, eb, bits, op)
    N = self.world
    out = torch.empty_like(x) if out is None else out
    self.ws.reset_status()
    self._copy_checked(x, out, reset=False)  # out is the working buffer (acc), input checked
    if N > 1:
        spans = chunk_spans(x.numel(), N)
        m = max(hi - lo for lo, hi in spans)
        _setup(self, codec, m, bits)
        ring = _Ring(self, codec, ebf, bits, op)
        _reduce_scatter_into(ring, out, spans)
        _allgather_owned(ring, out, spans, lambda j: (j + 1) % N)
        ring.done()
    if check:
        self.check()
    return out


def generic_reduce_scatter(self, x: torch.Tensor, codec: str = "none", eb: float | None = None, bits: int = 8,
                           op: str = "sum", check: bool = True):
    """ring_reduce_scatter_c with verbatim / fixed-rate messages: returns chunk (rank + 1) mod N."""
    x, ebf, bits = _prepare(self, x, codec, eb, bits, op)
    N, i = self.world, self.rank
    work = torch.empty_like(x)
    self.ws.reset_status()
    self._copy_checked(x, work, reset=False)
    spans = chunk_spans(x.numel(), N)
    if N > 1:
        _setup(self, codec, max(hi - lo for lo, hi in spans), bits)
        ring = _Ring(self, codec, ebf, bits, op)
        _reduce_scatter_into(ring, work, spans)
        ring.done()
    lo, hi = spans[(i + 1) % N]
    res = work[lo:hi].clone()
    if check:
        self.check()
    return res


def generic_allgather(self, chunk: torch.Tensor, codec: str = "none", eb: float | None = None, bits: int = 8,
                      check: bool = True):
    """ring_allgather_c (allgatherv) with verbatim / fixed-rate / per-hop messages:
    codec "none" / "fixed-rate" encode once at the owner (collectives.py:247-255);
    use :func:`cprp2p_allgather` for the compress-per-hop baseline."""
    chunk, ebf, bits = _prepare(self, chunk, codec, eb, bits, "sum")
    N, i = self.world, self.rank
    counts = [None] * N
    dist.all_gather_object(counts, int(chunk.numel()), group=self.group)
    lo = [0]
    for c_ in counts:
        lo.append(lo[-1] + c_)
    spans = [(lo[r], lo[r + 1]) for r in range(N)]
    out = torch.empty(lo[-1], dtype=torch.float32, device=self.device)
    self.ws.reset_status()
    self._copy_checked(chunk, out[spans[i][0]:spans[i][1]], reset=False)
    if N > 1:
        _setup(self, codec, max(counts), bits)
        ring = _Ring(self, codec, ebf, bits, "sum")
        _allgather_owned(ring, out, spans, lambda j: j)
        ring.done()
    if check:
        self.check()
    return out


def cprp2p_allgather(self, chunk: torch.Tensor, eb: float, check: bool = True):
    """cprp2p_allgather (collectives.py:311-341): the compress-per-hop baseline.
    At hop s rank i compresses the chunk it received at hop s-1 (its own at
    s = 0) and its right neighbour decodes it: a chunk that travelled h hops
    carries up to h * eb of error.  Chunks may differ in length."""
    chunk, ebf, _ = _prepare(self, chunk, "ebz", eb, 8, "sum")
    N, i = self.world, self.rank
    counts = [None] * N
    dist.all_gather_object(counts, int(chunk.numel()), group=self.group)
    lo = [0]
    for c_ in counts:
        lo.append(lo[-1] + c_)
    out = torch.empty(lo[-1], dtype=torch.float32, device=self.device)
    self.ws.reset_status()
    self._copy_checked(chunk, out[lo[i]:lo[i + 1]], reset=False)
    if N > 1:
        _setup(self, "ebz", max(counts), 8)
        ring = _Ring(self, "ebz", ebf, 8, "sum")
        right, left = (i + 1) % N, (i - 1) % N
        cur = i
        for s in range(N - 1):
            ring.send(s, out[lo[cur]:lo[cur + 1]], [right])
            cur = (i - 1 - s) % N
            ring.recv(s, left, out[lo[cur]:lo[cur + 1]], reduce=False)
        ring.done()
    if check:
        self.check()
    return out


Communicator.generic_allreduce = generic_allreduce
Communicator.generic_reduce_scatter = generic_reduce_scatter
Communicator.generic_allgather = generic_allgather
Communicator.cprp2p_allgather = cprp2p_allgather
Communicator.lossless_allreduce = lambda self, x, op="sum", out=None, check=True: generic_allreduce(
    self, x, "none", op=op, out=out, check=check)
Communicator.lossless_reduce_scatter = lambda self, x, op="sum", check=True: generic_reduce_scatter(
    self, x, "none", op=op, check=check)
Communicator.lossless_allgather = lambda self, chunk, check=True: generic_allgather(self, chunk, "none", check=check)
Communicator.fixed_rate_allreduce = lambda self, x, bits=8, op="sum", out=None, check=True: generic_allreduce(
    self, x, "fixed-rate", bits=bits, op=op, out=out, check=check)
