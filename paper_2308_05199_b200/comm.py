"""Compressed collectives across GPUs: one process per GPU over NVLink peer memory.

The per-rank schedules are the reference's (collectives.py:215-308,
349-424, 467-532); the simulated network (simnet.py) is replaced by CUDA-IPC
mapped buffers:

ring reduce-scatter (collectives.py:258-291)
    step 0   gz_compress(local chunk i)                  -> own out slot[0]
    step s   wait "left's slot[s] ready"; gz_reduce_step(left's slot[s] read
             over NVLink, local chunk (i-s-1) mod N)
             -> own out slot[s+1]   (s < N-2)
             -> own blob + owned f32 chunk (i+1) mod N (s = N-2)
    The fused kernel reads the left neighbour's blob straight out of its
    HBM (the loads overlap the decode/encode of other tiles).  Block offsets
    and widths travel in the sidecar, so no size message is needed (the size
    exchange is overlapped with compression, north_star).
compress-once allgather (collectives.py:215-244)
    the owner's blob is compressed once (the last RS step); every other rank
    pulls those bytes into a local landing slot on a side stream and decodes
    them while the next pull is in flight; the bytes are never recompressed,
    so the allreduce error stays <= N * eb.
recursive doubling (collectives.py:349-424) and binomial scatter (467-532)
    see Communicator.rd_allreduce / Communicator.binomial_scatter.

Synchronisation is stream-ordered (cuStreamWriteValue32 / WaitValue32 on
peer-mapped flag words): no host round trips, no spinning kernels.  The ring
flags are binary semaphores ("consumed" flags start free), so a repeated
call is captured once into a CUDA graph and replayed.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib as L
from .codec import Workspace, _check_eb
from .collectives import _check_op, chunk_spans, scatter_counts
from .schedule import Compress, Reduce, ring_allreduce_plan

_ALIGN = 256
_MAX_DECODE_SEGMENTS = 8  # GZ_MAX_DECODE_SEGMENTS (include/gzccl.h)
_NO_REPORT = (1 << 64) - 1  # gz_step_io.report_base: `local` is not the caller's input
_KEY_NONE = (1 << 63) - 1  # check(): no error on any rank
_KEY_MASK = (1 << 56) - 1
AG_COPY_SMS = 24  # SMs left to the allgather's NVLink pulls while the previous owner's blob is decoded
AG_MULTI_MAX = 8 << 20  # chunk values up to which the allgather decodes every owner in one remote-read launch


def _al(v: int) -> int:
    return (v + _ALIGN - 1) // _ALIGN * _ALIGN


class _Layout:
    """Carve one device buffer into flags, RS output slots, allgather landing
    slots and the owned blob."""

    def __init__(self, world: int, m_max: int):
        lib = L.lib()
        self.world = world
        self.blob_cap = _al(int(lib.gz_compress_bound(m_max)))
        self.sc_bytes = _al(int(lib.gz_sidecar_bytes(m_max)))
        # flags (u32): rs_full[world], ag_ready[world], rs_consumed[1], ag_consumed[world]
        self.flag_words = 3 * world + 1
        off = _al(4 * self.flag_words)
        self.len_off = off  # u64 lengths: slots[world] + own[1]
        off += _al(8 * (world + 1))
        # reduce-scatter outputs of this rank in slotted form (tile t at t * 4224,
        # sizes, widths), read in place by the right neighbour's fused step
        nt = int(lib.gz_num_tiles(m_max))
        self.slots_bytes = _al(int(lib.gz_slots_bytes(m_max)))
        self.slot_off = []
        for _ in range(max(world - 1, 0)):
            sl = off
            off += self.slots_bytes
            sz = off
            off += _al(4 * nt)
            wd = off
            off += _al(32 * nt)
            self.slot_off.append((sl, sz, wd))
        self.land_off = []  # allgather landing slots (owners' blobs pulled here)
        for _ in range(max(world - 1, 0)):
            self.land_off.append((off, off + self.blob_cap))
            off += self.blob_cap + self.sc_bytes
        self.own_off = (off, off + self.blob_cap)
        off += self.blob_cap + self.sc_bytes
        # the owned chunk's compress-once message in slotted form (ag_mode "slots"): the last
        # reduce-scatter step writes it without a gather, the peers decode it in place
        sl = off
        off += self.slots_bytes
        sz = off
        off += _al(4 * nt)
        wd = off
        off += _al(32 * nt)
        self.own_slot = (sl, sz, wd)
        self.total = off

    def rs_full(self, s):
        return 4 * s

    def ag_ready(self, j):
        return 4 * (self.world + j)

    def rs_consumed(self):
        return 4 * (2 * self.world)

    def ag_consumed(self, j):
        return 4 * (2 * self.world + 1 + j)


class Communicator:
    """One rank of a compressed-collective communicator (one process per GPU).

    ``group`` is a torch.distributed process group (NCCL or gloo) used only
    for the one-time exchange of IPC handles.
    """

    def __init__(self, group=None, device=None):
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ws = Workspace(self.device)  # status record + tile workspace of rd / scatter
        # the ring's own tile workspace: sized once per _setup, so the raw pointer a
        # captured ring graph holds can never be freed by another collective growing
        # its workspace (the graph cache is cleared whenever _setup reallocates)
        self._ring_ws = Workspace(self.device)
        self.flag_timeout_s = 60.0  # host-side bound on check()/synchronize() waits
        self.stream = torch.cuda.current_stream(self.device)
        self.epoch = 0
        self._n = None
        self._buf = None
        self._peer = None
        self.last_compression_ratio = None
        self.launches_per_call = 0
        self.events = None  # list -> (label, cuda event) marks after every wait/launch (profiling)
        self.stamps = None  # int64 device tensor -> %globaltimer stamps at the same marks (profiling)
        self.stamp_labels = []
        self.copy_stream = torch.cuda.Stream(self.device)  # allgather pulls
        self.use_graphs = True  # replay repeated ring calls from a captured CUDA graph
        self.graph_launches = 0  # kernels executed by graph replays (not seen by gz_launch_count)
        self.capture_stream = torch.cuda.Stream(self.device)
        self._graph_cache = {}
        self._last_key = None
        self._seen_keys = set()
        # allgather: "slots" (default: the owner's last reduce-scatter step leaves its message in slotted
        # form -- no gather kernel on the critical path -- and every peer decodes the owners' slots in
        # place over NVLink, one launch per 8 owners), or the blob-based modes: "multi" (one launch
        # decodes every owner's blob out of its memory), "copy" (pull each blob over NVLink on a side
        # stream, decode it locally) and "auto" (multi up to AG_MULTI_MAX values, copy above)
        self.ag_mode = "slots"
        # intermediate reduce-scatter steps take their input flag inside the kernel (one CTA
        # thread polls, bounded) instead of a stream wait node: ~5 µs less per step
        self.kernel_waits = True
        self.early_pull = False  # allreduce: allgather pulls start when each owner is ready, not after our last step

    # ------------------------------------------------------------------ setup
    def _setup(self, m_max: int):
        """(Re)build the IPC buffer for chunks of up to m_max values."""
        if self._n is not None and self._n >= m_max:
            return
        self._close()
        lib = L.lib()
        self.layout = _Layout(self.world, m_max)
        self._buf = torch.zeros(self.layout.total, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        hsz = lib.gz_ipc_handle_size()
        h = (ctypes.c_char * hsz)()
        L.check(lib.gz_ipc_get_handle(self._buf.data_ptr(), h), "gz_ipc_get_handle")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=self.group)
        self._peer = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                self._peer.append(self._buf.data_ptr())
            else:
                ptr = ctypes.c_void_p()
                L.check(lib.gz_ipc_open_handle(ctypes.create_string_buffer(hb, hsz), ctypes.byref(ptr)),
                        "gz_ipc_open_handle")
                self._peer.append(ptr.value)
        # consumed flags start "free" (1): the first call needs no special case
        flags = self._buf[: 4 * self.layout.flag_words].view(torch.int32)
        flags[self.layout.rs_consumed() // 4] = 1
        for j in range(self.world):
            flags[self.layout.ag_consumed(j) // 4] = 1
        self._ring_ws.tile_ws(int(lib.gz_workspace_bytes(m_max)))  # allocated (and zeroed) before any capture
        torch.cuda.synchronize(self.device)
        self._n = m_max
        self.epoch = 0
        self._graph_cache = {}
        self._last_key = None
        self._seen_keys = set()
        dist.barrier(group=self.group)

    def _close(self):
        if self._peer is not None:
            lib = L.lib()
            torch.cuda.synchronize(self.device)
            for r, p in enumerate(self._peer):
                if r != self.rank and p:
                    lib.gz_ipc_close(p)
        self._peer = None
        self._buf = None
        self._n = None
        self._graph_cache = {}
        self._last_key = None
        self._seen_keys = set()
        _scatter_close(self)
        _rd_close(self)

    def close(self):
        try:
            dist.barrier(group=self.group)
        except Exception:
            pass
        self._close()

    def __del__(self):
        try:
            self._close()
        except Exception:
            pass

    # --------------------------------------------------------------- helpers
    def _addr(self, r: int, off: int) -> int:
        return self._peer[r] + off

    def _signal(self, r: int, off: int, value: int, s: int):
        L.check(L.lib().gz_stream_write_u32(s, self._addr(r, off), value), "gz_stream_write_u32")

    def _wait(self, off: int, value: int, s: int):
        L.check(L.lib().gz_stream_wait_u32_geq(s, self._addr(self.rank, off), value), "gz_stream_wait_u32_geq")
        self._mark("wait")

    # ring flags are binary semaphores (constant values, so a call can be
    # captured in a CUDA graph and replayed): post = write 1 into the peer's
    # flag; take = wait for 1 on our own flag, then reset it to 0
    def _post(self, r: int, off: int, s: int):
        self._signal(r, off, 1, s)

    def _take(self, off: int, s: int):
        self._take_all([off], s)

    def _flag_ops(self, ops, s: int):
        """ops: [(kind, addr, value)], kind 0 = write, 1 = wait >= value; one
        stream memory-op batch (a single graph node)."""
        arr = (_FlagOp * len(ops))(*[_FlagOp(a, v, k) for k, a, v in ops])
        L.check(L.lib().gz_stream_flag_ops(s, arr, len(ops)), "gz_stream_flag_ops")

    def _take_all(self, offs, s: int, mark: bool = True):
        """take several of our own flags: wait for all, then reset all (one batch)"""
        mine = [self._addr(self.rank, off) for off in offs]
        self._flag_ops([(1, a, 1) for a in mine] + [(0, a, 0) for a in mine], s)
        if mark:
            self._mark("wait")

    def _post_all(self, targets, s: int):
        """post flags in several peers' memory: [(rank, off)] (one batch)"""
        self._flag_ops([(0, self._addr(r, off), 1) for r, off in targets], s)

    def _mark(self, label: str, stream: int | None = None):
        if self.stamps is not None:  # profiling: device timestamps, also inside a captured graph
            k = len(self.stamp_labels)
            if k < self.stamps.numel():
                self.stamp_labels.append(label)
                s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
                L.lib().gz_debug_stamp(self.stamps.data_ptr() + 8 * k, s)
        if self.events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(self.device))
            self.events.append((label, ev))

    # ------------------------------------------------------------ collectives
    def ring_allreduce(self, x: torch.Tensor, eb: float, op: str = "sum", out: torch.Tensor | None = None,
                       check: bool = True):
        """Per-rank ring_allreduce_c (collectives.py:294-308) on this GPU.

        Returns this rank's output: its own reduced chunk (i+1) mod N exact, all
        other chunks decoded from their owners' compress-once blobs.

        Errors (codec.py:79-86 / 273-322) are detected on the device by the
        kernels that read the data.  ``check=True`` waits for the call (bounded
        by ``flag_timeout_s``) and raises on every rank the error the reference
        would raise: ``ValueError("non-finite value at offset k")`` for the
        first bad value in rank order.  ``check=False`` leaves the call
        asynchronous; the next :meth:`check` reports its errors.
        """
        x = self._check_input(x)
        ebf, opc = _check_eb(eb), _check_op(op)
        if out is None:
            out = torch.empty_like(x)
        if self.world == 1:
            self._copy_checked(x, out)
        else:
            spans = chunk_spans(x.numel(), self.world)
            self._run_graphed("allreduce", x, spans, ebf, opc, out)
        if check:
            self.check()
        return out

    def _run_graphed(self, mode, x, spans, ebf, opc, out):
        """Run one ring collective; a call repeated on the same tensors and
        parameters is captured once into a CUDA graph and then replayed (one
        launch of the whole schedule: kernels, peer flags, the allgather's
        side-stream pulls), which removes the per-call host cost."""
        key = (mode, x.data_ptr(), x.numel(), out.data_ptr(), out.numel(), ebf, opc, self.ag_mode, self.kernel_waits, self.early_pull)
        if self.use_graphs and self.events is None and not torch.cuda.is_current_stream_capturing():
            g = self._graph_cache.get(key) if self._n is not None else None
            if g is not None:
                g[0].replay()
                self.graph_launches += g[1]
                self.launches_per_call = g[1]
                return
            if self._n is not None and key in self._seen_keys and len(self._graph_cache) < 16:
                g = torch.cuda.CUDAGraph()
                s0 = torch.cuda.current_stream(self.device)
                with torch.cuda.graph(g, stream=self.capture_stream):
                    self._ring(mode, x, spans, ebf, opc, out)
                s0.wait_stream(self.capture_stream)
                self._graph_cache[key] = (g, self.launches_per_call)
                g.replay()
                self.graph_launches += self.launches_per_call
                return
        self._last_key = key
        self._seen_keys.add(key)  # a second call with the same key is captured (also when keys alternate)
        self._ring(mode, x, spans, ebf, opc, out)

    def ring_reduce_scatter(self, x: torch.Tensor, eb: float, op: str = "sum", out: torch.Tensor | None = None,
                            check: bool = True):
        """Per-rank ring_reduce_scatter_c (collectives.py:258-291): returns the
        fully reduced chunk (rank + 1) mod N of chunk_spans(n, N).  The last step
        decodes and reduces without re-compressing (gz_decompress_reduce).
        ``check`` as in :meth:`ring_allreduce`."""
        x = self._check_input(x)
        ebf, opc = _check_eb(eb), _check_op(op)
        N, i = self.world, self.rank
        spans = chunk_spans(x.numel(), N)
        lo, hi = spans[(i + 1) % N]
        if out is None:
            out = torch.empty(hi - lo, dtype=torch.float32, device=self.device)
        if N == 1:
            self._copy_checked(x, out)
        else:
            self._run_graphed("reduce_scatter", x, spans, ebf, opc, out)
        if check:
            self.check()
        return out

    def ring_allgather(self, chunk: torch.Tensor, eb: float, out: torch.Tensor | None = None, check: bool = True):
        """Per-rank ring_allgather_c (collectives.py:247-255), allgatherv: every
        rank contributes a chunk of any length; each rank compresses its chunk
        once and the others decode those bytes; the own chunk is kept verbatim.
        Returns the concatenation in rank order.  ``check`` as in
        :meth:`ring_allreduce`."""
        chunk = self._check_input(chunk)
        ebf = _check_eb(eb)
        N = self.world
        counts = [None] * N
        dist.all_gather_object(counts, int(chunk.numel()), group=self.group)  # lengths ride in the headers
        total = sum(counts)
        if out is None:
            out = torch.empty(total, dtype=torch.float32, device=self.device)
        if N == 1:
            self._copy_checked(chunk, out)
        else:
            lo = [0]
            for c in counts:
                lo.append(lo[-1] + c)
            spans = [(lo[r], lo[r + 1]) for r in range(N)]
            self._ring("allgather", chunk, spans, ebf, 0, out)
        if check:
            self.check()
        return out

    # ------------------------------------------------------------ errors
    def _copy_checked(self, src: torch.Tensor, dst: torch.Tensor, report_base: int = 0, reset: bool = True):
        """dst = src on the device, recording the first non-finite offset."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        if reset:
            self.ws.reset_status()
        if src.numel():
            L.check(L.lib().gz_copy_checked(src.data_ptr(), dst.data_ptr(), src.numel(), report_base,
                                            self.ws.status_ptr(), s), "gz_copy_checked")

    def _bounded_sync(self, what: str = "collective"):
        """Wait for this rank's stream, at most ``flag_timeout_s`` seconds.  A
        peer that never posts its flag leaves a stream-ordered wait pending
        forever: the flags of our buffers are then forced (from a side stream)
        so the queued work drains, the communicator is marked broken and
        TimeoutError is raised instead of hanging the process."""
        import time

        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        t0 = time.perf_counter()
        # spin for the first 2 ms (a collective usually ends within that:
        # sleeping would add the scheduler's wake-up latency to every call),
        # then back off
        while not ev.query():
            waited = time.perf_counter() - t0
            if waited > self.flag_timeout_s:
                self._poison()
                raise TimeoutError(f"rank {self.rank}: {what} did not complete within {self.flag_timeout_s} s "
                                   "(a peer never posted its flag); the communicator is unusable")
            if waited > 2e-3:
                time.sleep(min(1e-2, waited / 8))

    def _poison(self):
        side = torch.cuda.Stream(self.device)
        with torch.cuda.stream(side):
            for buf in (self._buf, getattr(self, "_sc_buf", None), getattr(self, "_rd_buf", None)):
                if buf is not None:
                    nflag = 4 * 64  # every flag area is at the start of its buffer
                    buf[: min(nflag, buf.numel())].view(torch.int32).fill_(0x3FFFFFFF)
        self._broken = True

    def check(self):
        """Wait for the outstanding calls of this rank (bounded) and raise the
        first error any rank's kernels recorded since the last reset, on every
        rank alike (the reference raises for the whole collective).  The ranks'
        status words are combined on the device (one MIN all-reduce of
        (rank << 56 | value) keys, so the lowest rank with an error wins, as in
        collectives.py:202-205), then read with one small copy."""
        from .codec import DecodeError

        if getattr(self, "_broken", False):
            raise RuntimeError("communicator is unusable after a peer timeout")
        if not hasattr(self, "_st_key"):
            self._st_key = torch.empty(4, dtype=torch.int64, device=self.device)
        key = self._st_key
        L.check(L.lib().gz_status_key(self.ws.status_ptr(), self.rank, key.data_ptr(),
                                      torch.cuda.current_stream(self.device).cuda_stream), "gz_status_key")
        if self.world > 1:
            dist.all_reduce(key, op=dist.ReduceOp.MIN, group=self.group)
        if not hasattr(self, "_st_host"):
            self._st_host = torch.empty(4, dtype=torch.int64, pin_memory=True)
        self._st_host.copy_(key, non_blocking=True)
        self._bounded_sync()
        k = [int(v) for v in self._st_host.tolist()]
        if k[3] != _KEY_NONE:
            raise RuntimeError(f"rank {k[3] >> 56}: a peer flag never arrived (in-kernel wait gave up after 20 s)")
        if k[0] != _KEY_NONE:
            raise ValueError(f"non-finite value at offset {k[0] & _KEY_MASK}")
        if k[1] != _KEY_NONE:
            e = k[1] & _KEY_MASK
            raise DecodeError(f"rank {k[1] >> 56}: inconsistent compressed stream at block {e >> 24} (code {e & 0xFF})")

    def _check_input(self, x):
        if not isinstance(x, torch.Tensor) or x.dim() != 1 or x.dtype != torch.float32 or not x.is_cuda:
            raise ValueError("expected a flat 1-D float32 CUDA tensor")
        return x.contiguous()

    def _ring(self, mode: str, x, spans, ebf: float, opc: int, out):
        """Shared executor.  mode: "allreduce" (RS + compress-once AG),
        "reduce_scatter" (RS only), "allgather" (compress own chunk + AG).
        spans: per-chunk [lo, hi) (chunk_spans, or the allgatherv layout)."""
        N, i = self.world, self.rank
        m_max = max(hi - lo for lo, hi in spans)
        self._setup(m_max)
        lib = L.lib()
        lay = self.layout
        cur = torch.cuda.current_stream(self.device)  # (a capture stream while recording a graph)
        s = cur.cuda_stream
        ws = self.ws
        tws = self._ring_ws.tile_ws(int(lib.gz_workspace_bytes(m_max)))  # no reallocation: sized in _setup
        ws.reset_status(cur)  # errors of this call only (a memset node when captured)
        e = self.epoch + 1
        right, left = (i + 1) % N, (i - 1) % N
        self.spans = spans

        def chunk_ptr(t, c):
            return t.data_ptr() + 4 * spans[c][0]

        def msize(c):
            return spans[c][1] - spans[c][0]

        def slot(r, k):  # (slots, sizes, widths) of rank r's reduce-scatter output k
            sl, sz, wd = lay.slot_off[k]
            return self._addr(r, sl), self._addr(r, sz), self._addr(r, wd)

        def step(inp, local, n_, acc, out_slot=None, out_blob=None, post=None, wait=None, base=0):
            io = _StepIO()
            io.report_base = base  # offset of `local` in x: non-finite inputs are reported like codec.py:79-86
            if inp is not None:
                io.in_slots, io.in_sizes, io.in_widths = inp
            if out_slot is not None:
                io.out_slots, io.out_sizes, io.out_widths = out_slot
                if post is not None:  # the kernel posts the peer's flag itself when done
                    io.post_flag = self._addr(*post)
                if wait is not None:  # ... and takes our own flag itself before reading
                    io.wait_flag = self._addr(i, wait)
            else:
                io.blob_out, io.blob_out_cap, io.d_len_out, io.sidecar_out = out_blob
            L.check(lib.gz_step(ctypes.byref(io), local, n_, ebf, opc, acc, tws.data_ptr(), tws.numel(),
                                ws.status_ptr(), s), "gz_step")

        own_free = None
        if mode == "allreduce":
            # peers must have consumed our previous own blob before the last RS
            # step rewrites it: waited for on a side branch, off the ring's
            # critical path (joined just before that step)
            fork = torch.cuda.Event()
            fork.record(cur)
            self.copy_stream.wait_event(fork)
            self._take_all([lay.ag_consumed(j) for j in range(N) if j != i], self.copy_stream.cuda_stream, False)
            own_free = torch.cuda.Event()
            own_free.record(self.copy_stream)

        def wait_own_blob_free():
            if own_free is not None:
                cur.wait_event(own_free)
            else:
                self._take_all([lay.ag_consumed(j) for j in range(N) if j != i], s)

        def own_ready():
            self._post_all([(j, lay.ag_ready(i)) for j in range(N) if j != i], s)

        launches = 0
        self.stamp_labels = []
        self._mark("start")
        if mode in ("allreduce", "reduce_scatter"):
            # the right neighbour must have consumed our previous writes (taken
            # inside the first step kernel, like every intermediate step's input flag)
            if not self.kernel_waits:
                self._take(lay.rs_consumed(), s)
            for p in ring_allreduce_plan(N, i):
                if isinstance(p, Compress):
                    # step 0: compress the local chunk into our output slot 0 (slotted: no
                    # gather); the right neighbour's fused step reads it in place
                    step(None, chunk_ptr(x, p.chunk), msize(p.chunk), None, out_slot=slot(i, p.slot),
                         post=(p.dst, lay.rs_full(p.slot)),
                         wait=lay.rs_consumed() if self.kernel_waits else None, base=spans[p.chunk][0])
                    launches += 1
                    self._mark("compress")
                elif isinstance(p, Reduce):
                    if p.last or not self.kernel_waits:
                        self._take(lay.rs_full(p.slot), s)
                    inp = slot(left, p.slot)  # the left neighbour's output, read over NVLink
                    if p.last and mode == "reduce_scatter":
                        # decode + reduce into the owned chunk; nothing to re-compress
                        io = _StepIO()
                        io.in_slots, io.in_sizes, io.in_widths = inp
                        io.report_base = spans[p.chunk][0]
                        L.check(lib.gz_step_reduce(ctypes.byref(io), chunk_ptr(x, p.chunk), msize(p.chunk), ebf,
                                                   opc, out.data_ptr(), ws.status_ptr(), s), "gz_step_reduce")
                        launches += 1
                        self._mark("reduce_last")
                        continue
                    # fused decompress(recv) + op + compress
                    if not p.last:
                        step(inp, chunk_ptr(x, p.chunk), msize(p.chunk), None, out_slot=slot(i, p.slot + 1),
                             post=(p.dst, lay.rs_full(p.slot + 1)),
                             wait=lay.rs_full(p.slot) if self.kernel_waits else None, base=spans[p.chunk][0])
                        launches += 1
                    elif self.ag_mode == "slots":
                        wait_own_blob_free()  # our own message is read by every peer in the allgather
                        step(inp, chunk_ptr(x, p.chunk), msize(p.chunk), chunk_ptr(out, p.chunk),
                             out_slot=tuple(self._addr(i, o) for o in lay.own_slot), base=spans[p.chunk][0])
                        launches += 1
                    else:
                        wait_own_blob_free()  # our own blob is read by every peer in the allgather
                        step(inp, chunk_ptr(x, p.chunk), msize(p.chunk), chunk_ptr(out, p.chunk),
                             out_blob=(self._addr(i, lay.own_off[0]), lay.blob_cap,
                                       self._addr(i, lay.len_off + 8 * N), self._addr(i, lay.own_off[1])),
                             base=spans[p.chunk][0])
                        launches += 2
                    self._mark("reduce_last" if p.last else "reduce")
                    if p.last:
                        own_ready()
        if mode == "allgather":
            # compress our chunk once into our own blob; the own chunk is kept verbatim
            wait_own_blob_free()
            if self.ag_mode == "slots":
                step(None, x.data_ptr(), x.numel(), None, out_slot=tuple(self._addr(i, o) for o in lay.own_slot))
                launches += 1
            else:
                L.check(lib.gz_compress(x.data_ptr(), x.numel(), ebf, 32, self._addr(i, lay.own_off[0]), lay.blob_cap,
                                        self._addr(i, lay.len_off + 8 * N), self._addr(i, lay.own_off[1]), None,
                                        tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_compress")
                launches += 2
            self._mark("compress")
            own_ready()
            if x.numel():
                out[spans[i][0]:spans[i][1]].copy_(x)
        if mode in ("allreduce", "allgather"):
            # compress-once allgather; owner j's chunk is chunk_of(j)
            owners = [(i - 1 - k) % N for k in range(N - 1)]  # the order the ring delivers them
            chunk_of = (lambda j: (j + 1) % N) if mode == "allreduce" else (lambda j: j)
            launches += self._allgather_pull(owners, chunk_of, chunk_ptr, msize, out, ebf, cur,
                                             forked=own_free is not None)
        # our slots are free again: the left neighbour may write the next call's steps
        self._post(left, lay.rs_consumed(), s)
        self.epoch = e
        self.launches_per_call = launches

    def _allgather_pull(self, owners, chunk_of, chunk_ptr, msize, out, ebf, cur, forked=False) -> int:
        """A side stream pulls each owner's blob + sidecar over NVLink into our
        (free) reduce-scatter slots with one bulk copy and releases the owner;
        the main stream decodes it from local HBM as soon as it has landed,
        while the next copy is in flight.  A single owner (N = 2) is decoded
        straight out of its memory."""
        lib = L.lib()
        lay = self.layout
        N, i = self.world, self.rank
        s = cur.cuda_stream
        ws = self.ws
        launches = 0
        mode = self.ag_mode
        if mode == "slots":
            # every owner's slotted message decoded in place (peer memory), 8 owners per launch
            self._take_all([lay.ag_ready(j) for j in owners], s)
            nl = 0
            for g0 in range(0, len(owners), _MAX_DECODE_SEGMENTS):
                grp = owners[g0:g0 + _MAX_DECODE_SEGMENTS]
                k = len(grp)
                P = ctypes.c_void_p * k
                sls = P(*[self._addr(j, lay.own_slot[0]) for j in grp])
                szs = P(*[self._addr(j, lay.own_slot[1]) for j in grp])
                wds = P(*[self._addr(j, lay.own_slot[2]) for j in grp])
                ns = (ctypes.c_uint64 * k)(*[msize(chunk_of(j)) for j in grp])
                ys = P(*[chunk_ptr(out, chunk_of(j)) for j in grp])
                L.check(lib.gz_decompress_slots_multi(sls, szs, wds, ns, k, ebf, ys, 0, ws.status_ptr(), s),
                        "gz_decompress_slots_multi")
                nl += 1
            self._mark("decode")
            self._post_all([(j, lay.ag_consumed(i)) for j in owners], s)
            return nl
        if mode == "auto":
            mode = "multi" if max(msize(chunk_of(j)) for j in owners) <= AG_MULTI_MAX else "copy"
        if len(owners) > 1 and mode == "multi":
            # one launch decodes every owner's blob straight out of its memory
            self._take_all([lay.ag_ready(j) for j in owners], s)
            nl = 0
            for g0 in range(0, len(owners), _MAX_DECODE_SEGMENTS):  # one launch per 8 owners
                grp = owners[g0:g0 + _MAX_DECODE_SEGMENTS]
                k = len(grp)
                P = ctypes.c_void_p * k
                blobs = P(*[self._addr(j, lay.own_off[0]) for j in grp])
                scs = P(*[self._addr(j, lay.own_off[1]) for j in grp])
                ns = (ctypes.c_uint64 * k)(*[msize(chunk_of(j)) for j in grp])
                ys = P(*[chunk_ptr(out, chunk_of(j)) for j in grp])
                L.check(lib.gz_decompress_multi(blobs, scs, ns, k, ebf, ys, 0, ws.status_ptr(), s),
                        "gz_decompress_multi")
                nl += 1
            self._mark("decode")
            self._post_all([(j, lay.ag_consumed(i)) for j in owners], s)
            return nl
        if mode == "bulk" and len(owners) > _MAX_DECODE_SEGMENTS:
            mode = "copy"
        if mode == "bulk":
            # pull every owner's blob + sidecar in ONE copy launch (the NVLink ingress is the
            # bound; a decode beside a pull runs barely faster than after it), then decode
            # them all from local HBM in one launch
            self._take_all([lay.ag_ready(j) for j in owners], s)
            items = []
            for k, j in enumerate(owners):
                b, sc = lay.land_off[k]
                items.append(_CopyItem(self._addr(j, lay.own_off[0]), self._addr(i, b), self._addr(j, lay.len_off + 8 * N),
                                       lay.blob_cap))
                items.append(_CopyItem(self._addr(j, lay.own_off[1]), self._addr(i, sc), None,
                                       int(lib.gz_sidecar_bytes(msize(chunk_of(j))))))
            L.check(lib.gz_copy_items_sms((_CopyItem * len(items))(*items), len(items), 0, s), "gz_copy_items_sms")
            self._mark("copy")
            self._post_all([(j, lay.ag_consumed(i)) for j in owners], s)
            k = len(owners)
            P = ctypes.c_void_p * k
            blobs = P(*[self._addr(i, lay.land_off[q][0]) for q in range(k)])
            scs = P(*[self._addr(i, lay.land_off[q][1]) for q in range(k)])
            ns = (ctypes.c_uint64 * k)(*[msize(chunk_of(j)) for j in owners])
            ys = P(*[chunk_ptr(out, chunk_of(j)) for j in owners])
            L.check(lib.gz_decompress_multi(blobs, scs, ns, k, ebf, ys, 0, ws.status_ptr(), s), "gz_decompress_multi")
            self._mark("decode")
            return 2
        if len(owners) == 1 and mode != "copy":  # N = 2, small chunk: decode straight from the peer
            j = owners[0]
            c = chunk_of(j)
            self._take(lay.ag_ready(j), s)
            L.check(lib.gz_decompress_sidecar(self._addr(j, lay.own_off[0]), self._addr(j, lay.own_off[1]), msize(c),
                                              ebf, chunk_ptr(out, c), ws.status_ptr(), s), "gz_decompress_sidecar")
            self._mark("decode")
            self._post(j, lay.ag_consumed(i), s)
            return 1
        cs = self.copy_stream.cuda_stream
        if not forked or not self.early_pull:
            # the landing slots are free once the previous call's decodes are done:
            # the allreduce's side stream is already ordered after them (forked at
            # the call's start), so its pulls start as soon as each owner is ready
            rs_done = torch.cuda.Event()
            rs_done.record(cur)
            self.copy_stream.wait_event(rs_done)
        landed = []
        for k, j in enumerate(owners):
            self._take_all([lay.ag_ready(j)], cs, False)
            b, sc = lay.land_off[k]
            items = (_CopyItem * 2)(
                _CopyItem(self._addr(j, lay.own_off[0]), self._addr(i, b), self._addr(j, lay.len_off + 8 * N),
                          lay.blob_cap),
                _CopyItem(self._addr(j, lay.own_off[1]), self._addr(i, sc), None,
                          int(lib.gz_sidecar_bytes(msize(chunk_of(j))))))
            # the first pull has the GPU to itself; later ones run beside a decode
            L.check(lib.gz_copy_items_sms(items, 2, AG_COPY_SMS if k else 0, cs), "gz_copy_items_sms")
            launches += 1
            self._mark("copy", cs)
            self._post(j, lay.ag_consumed(i), cs)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
            landed.append(ev)
        for k, j in enumerate(owners):
            c = chunk_of(j)
            cur.wait_event(landed[k])
            b, sc = lay.land_off[k]
            P = ctypes.c_void_p * 1
            L.check(lib.gz_decompress_multi(P(self._addr(i, b)), P(self._addr(i, sc)), (ctypes.c_uint64 * 1)(msize(c)), 1,
                                            ebf, P(chunk_ptr(out, c)), AG_COPY_SMS if k + 1 < len(owners) else 0,
                                            ws.status_ptr(), s), "gz_decompress_multi")
            launches += 1
            self._mark("decode")
        return launches

    def compression_ratio(self) -> float:
        """Compressed size of this rank's owned chunk (last call), as a ratio."""
        lay = self.layout
        torch.cuda.synchronize(self.device)
        i = self.rank
        c = (i + 1) % self.world
        m = self.spans[c][1] - self.spans[c][0]
        if self.ag_mode == "slots":  # the owned message's tile sizes
            nt = int(L.lib().gz_num_tiles(m))
            sz = self._buf[lay.own_slot[1]:lay.own_slot[1] + 4 * nt].view(torch.int32)
            ln = int(sz.sum().item()) + 24  # the reference blob = header + payload
        else:
            ln = self._buf[lay.len_off + 8 * self.world : lay.len_off + 8 * self.world + 8].view(torch.int64).item()
        self.last_compression_ratio = round(4 * m / ln, 4) if ln else None
        return self.last_compression_ratio



class _StepIO(ctypes.Structure):  # gz_step_io (include/gzccl.h)
    _fields_ = [("in_blob", ctypes.c_void_p), ("in_sidecar", ctypes.c_void_p), ("in_slots", ctypes.c_void_p),
                ("in_sizes", ctypes.c_void_p), ("in_widths", ctypes.c_void_p), ("blob_out", ctypes.c_void_p),
                ("blob_out_cap", ctypes.c_uint64), ("d_len_out", ctypes.c_void_p), ("sidecar_out", ctypes.c_void_p),
                ("out_slots", ctypes.c_void_p), ("out_sizes", ctypes.c_void_p), ("out_widths", ctypes.c_void_p),
                ("post_flag", ctypes.c_void_p), ("wait_flag", ctypes.c_void_p), ("report_base", ctypes.c_uint64)]


class _FlagOp(ctypes.Structure):  # gz_flag_op (include/gzccl.h)
    _fields_ = [("ptr", ctypes.c_void_p), ("value", ctypes.c_uint32), ("kind", ctypes.c_uint32)]


class _CopyItem(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("d_len", ctypes.c_void_p),
                ("max_bytes", ctypes.c_uint64)]


class _ScatterLayout:
    """One IPC buffer per rank, same layout everywhere: flags, lengths, and a
    worst-case slot (blob + sidecar) per VIRTUAL rank, so a tree hop's range
    [lo, hi) is the same offsets on the parent and the child."""

    def __init__(self, world: int, vcounts):
        lib = L.lib()
        self.world = world
        off = _al(4 * (1 + world))  # u32 flags: ready, consumed[world]
        self.len_off = off
        off += _al(8 * world)
        self.slot, self.sc, self.cap, self.sc_bytes = [], [], [], []
        for c in vcounts:
            self.slot.append(off)
            self.cap.append(int(lib.gz_compress_bound(c)))
            off += _al(self.cap[-1])
            self.sc.append(off)
            self.sc_bytes.append(int(lib.gz_sidecar_bytes(c)))
            off += _al(self.sc_bytes[-1])
        self.total = off

    READY = 0

    @staticmethod
    def consumed(j):
        return 4 * (1 + j)


def _open_peers(comm, buf):
    lib = L.lib()
    hsz = lib.gz_ipc_handle_size()
    h = (ctypes.c_char * hsz)()
    L.check(lib.gz_ipc_get_handle(buf.data_ptr(), h), "gz_ipc_get_handle")
    handles = [None] * comm.world
    dist.all_gather_object(handles, bytes(h), group=comm.group)
    peers = []
    for r, hb in enumerate(handles):
        if r == comm.rank:
            peers.append(buf.data_ptr())
        else:
            ptr = ctypes.c_void_p()
            L.check(lib.gz_ipc_open_handle(ctypes.create_string_buffer(hb, hsz), ctypes.byref(ptr)), "gz_ipc_open_handle")
            peers.append(ptr.value)
    return peers


def _scatter_close(self):
    peers = getattr(self, "_sc_peer", None)
    if peers is not None:
        lib = L.lib()
        torch.cuda.synchronize(self.device)
        for r, p in enumerate(peers):
            if r != self.rank and p:
                lib.gz_ipc_close(p)
    self._sc_peer = None
    self._sc_buf = None
    self._sc_key = None


def binomial_scatter(self, x, eb: float, counts=None, root: int = 0, routing: str = "tree", out=None,
                     check: bool = True):
    """This rank's part of binomial_scatter_c (collectives.py:467-532).

    The root passes its whole buffer ``x`` (other ranks: None); every rank
    returns its ``counts[rank]`` values — the root its slice verbatim, the
    others their block decoded from the root's compress-once blob.

    * the root compresses the N-1 blocks it sends, in virtual-rank order, in
      ONE launch (gz_compress_segments = compress_blocks, codec.py:408-427);
      its own block, kept verbatim, is never sent, so it is not compressed;
    * routing="tree": each rank pulls its subtree's range [vr, vr+extent) of
      blobs + sidecars + lengths from its tree parent in one gz_copy_items
      launch (the reference's byte-range forwarding, collectives.py:511-525),
      then signals its children; routing="direct": every rank decodes its blob
      straight out of the root's memory (same bytes, same output — on NVSwitch
      all peers are one hop away);
    * the size table never travels separately: lengths sit next to the blobs
      and the sidecar carries the block offsets;
    * errors as in :meth:`Communicator.ring_allreduce` (``check``): a
      non-finite root value is reported with its offset in the root buffer.
    """
    from .schedule import scatter_route

    if routing not in ("tree", "direct"):
        raise ValueError(f"unknown routing {routing!r}")
    ebf = _check_eb(eb)
    N, me = self.world, self.rank
    if not 0 <= root < N:
        raise ValueError(f"root {root} out of range [0, {N})")
    meta = None
    if me == root:
        # validated at the root, the verdict broadcast so every rank raises alike
        try:
            if not isinstance(x, torch.Tensor) or x.dim() != 1 or x.dtype != torch.float32 or not x.is_cuda:
                raise ValueError("root buffer must be a flat 1-D float32 CUDA tensor")
            meta = [int(x.numel())] + scatter_counts(int(x.numel()), N, counts)
        except ValueError as err:
            meta = str(err)
    box = [meta]
    dist.broadcast_object_list(box, src=root, group=self.group)
    if isinstance(box[0], str):
        raise ValueError(box[0])
    n, counts = box[0][0], box[0][1:]
    if out is None:
        out = torch.empty(counts[me], dtype=torch.float32, device=self.device)
    lib = L.lib()
    s = self.stream.cuda_stream
    self.ws.reset_status()
    if N == 1:
        self._copy_checked(x, out, reset=False)
        self.launches_per_call = 1
        if check:
            self.check()
        return out
    order = [(root + j) % N for j in range(N)]  # virtual rank -> actual rank
    vcounts = [counts[order[v]] for v in range(N)]
    key = (n, tuple(counts), root, routing)
    if getattr(self, "_sc_key", None) != key:
        _scatter_close(self)
        self._sc_layout = _ScatterLayout(N, vcounts)
        self._sc_buf = torch.zeros(self._sc_layout.total, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        self._sc_peer = _open_peers(self, self._sc_buf)
        self._sc_key = key
        self._sc_epoch = 0
        dist.barrier(group=self.group)
    lay, peer = self._sc_layout, self._sc_peer
    prev, e = self._sc_epoch, self._sc_epoch + 1
    vr = (me - root) % N
    parent, _, sends = scatter_route(N, root)[me]
    launches = 0

    def at(r, off):
        return peer[r] + off

    if me == root:
        # blobs of the previous call must be consumed before they are overwritten
        if prev:
            for j in ([c for c, _, _ in sends] if routing == "tree" else [j for j in range(N) if j != me]):
                L.check(lib.gz_stream_wait_u32_geq(s, at(me, lay.consumed(j)), prev), "gz_stream_wait_u32_geq")
        lo = [0]
        for c in counts:
            lo.append(lo[-1] + c)
        # the root's own block (virtual rank 0) is never sent (root_sends cover
        # [1, N), collectives.py:503-508): only blocks 1..N-1 are compressed
        xv = x[lo[1]:] if root == 0 else torch.cat([x[lo[r]:lo[r + 1]] for r in order[1:]])
        arr = ctypes.c_uint64 * (N - 1)
        h_counts = arr(*vcounts[1:])
        ws = self.ws.tile_ws(int(lib.gz_segments_workspace_bytes(h_counts, N - 1)))
        base = self._sc_buf.data_ptr()
        L.check(lib.gz_compress_segments(xv.data_ptr(), h_counts, N - 1, ebf, base, arr(*lay.slot[1:]),
                                         base + lay.len_off + 8, base, arr(*lay.sc[1:]),
                                         arr(*[lo[order[v]] for v in range(1, N)]), ws.data_ptr(), ws.numel(),
                                         self.ws.status_ptr(), s), "gz_compress_segments")
        self._copy_checked(x[lo[me]:lo[me + 1]], out, report_base=lo[me], reset=False)
        launches += 2 + (root != 0)
        targets = [c for c, _, _ in sends] if routing == "tree" else [j for j in range(N) if j != me]
        for j in targets:
            L.check(lib.gz_stream_write_u32(s, at(j, lay.READY), e), "gz_stream_write_u32")
    else:
        L.check(lib.gz_stream_wait_u32_geq(s, at(me, lay.READY), e), "gz_stream_wait_u32_geq")
        if routing == "tree":
            # my children must be done with my previous range before I overwrite it
            if prev:
                for c, _, _ in sends:
                    L.check(lib.gz_stream_wait_u32_geq(s, at(me, lay.consumed(c)), prev), "gz_stream_wait_u32_geq")
            hi = max([h for _, _, h in sends], default=vr + 1)
            items = [_CopyItem(at(parent, lay.len_off + 8 * vr), at(me, lay.len_off + 8 * vr), None, 8 * (hi - vr))]
            for v in range(vr, hi):
                items.append(_CopyItem(at(parent, lay.slot[v]), at(me, lay.slot[v]), at(parent, lay.len_off + 8 * v),
                                       lay.cap[v]))
                items.append(_CopyItem(at(parent, lay.sc[v]), at(me, lay.sc[v]), None, lay.sc_bytes[v]))
            for k in range(0, len(items), 64):
                chunk = items[k:k + 64]
                L.check(lib.gz_copy_items((_CopyItem * len(chunk))(*chunk), len(chunk), s), "gz_copy_items")
                launches += 1
            # parent's range has been read: release it, then wake my children
            L.check(lib.gz_stream_write_u32(s, at(parent, lay.consumed(me)), e), "gz_stream_write_u32")
            for c, _, _ in sends:
                L.check(lib.gz_stream_write_u32(s, at(c, lay.READY), e), "gz_stream_write_u32")
            src = me
        else:
            src = root
        L.check(lib.gz_decompress_sidecar(at(src, lay.slot[vr]), at(src, lay.sc[vr]), counts[me], ebf, out.data_ptr(),
                                          self.ws.status_ptr(), s), "gz_decompress_sidecar")
        launches += 1
        if routing == "direct":
            L.check(lib.gz_stream_write_u32(s, at(root, lay.consumed(me)), e), "gz_stream_write_u32")
    self._sc_epoch = e
    self.launches_per_call = launches
    if check:
        self.check()
    return out


Communicator.binomial_scatter = binomial_scatter


class _RDLayout:
    """Recursive doubling: one slotted message buffer per message a rank can
    SEND -- 0: the donor's buffer (donors), 1..steps: the exchange steps,
    steps+1: the absorber's final result (absorbers) -- read in place by the
    receiving peer over NVLink; plus full[k] / consumed[k] flags."""

    def __init__(self, n: int, steps: int):
        lib = L.lib()
        self.K = steps + 2
        nt = int(lib.gz_num_tiles(n))
        off = _al(4 * 2 * self.K)
        self.slot = []
        for _ in range(self.K):
            sl = off
            off += _al(int(lib.gz_slots_bytes(n)))
            sz = off
            off += _al(4 * nt)
            wd = off
            off += _al(32 * nt)
            self.slot.append((sl, sz, wd))
        self.total = off

    def full(self, k):
        return 4 * k

    def consumed(self, k):
        return 4 * (self.K + k)


def rd_allreduce(self, x, eb: float, op: str = "sum", out=None, check: bool = True):
    """This rank's part of rd_allreduce_c (collectives.py:349-424) over NVLink.

    Whole-buffer exchanges with the partner actual(remapped(i) ^ 2^t).  Every
    message stays in the sender's memory in slotted form and the receiver's
    kernel reads it in place (pull); every reduction followed by a send is one
    fused kernel (decode the partner's message + op + compress), the last
    reduction of a non-absorber a decode+op kernel.  The input buffer is only
    read: the first reduction writes `out`.  Donors (even ranks below 2r) fold
    into their absorber first and receive the result compressed at the end.
    Outputs are per rank, bit-exact with the reference.
    """
    from .collectives import rd_plan

    x = self._check_input(x)
    ebf = _check_eb(eb)
    opc = _check_op(op)
    N, i = self.world, self.rank
    if out is None:
        out = torch.empty_like(x)
    self.ws.reset_status()
    if N == 1:
        self._copy_checked(x, out, reset=False)
        if check:
            self.check()
        return out
    n = x.numel()
    pof2, r, steps, role, remapped, actual = rd_plan(N)
    if getattr(self, "_rd_key", None) != (n, N):
        _rd_close(self)
        self._rd_layout = _RDLayout(n, steps)
        self._rd_buf = torch.zeros(self._rd_layout.total, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        self._rd_peer = _open_peers(self, self._rd_buf)
        self._rd_key = (n, N)
        self._rd_epoch = 0
        dist.barrier(group=self.group)
    lib = L.lib()
    lay, peer = self._rd_layout, self._rd_peer
    prev, e = self._rd_epoch, self._rd_epoch + 1
    s = self.stream.cuda_stream
    ws = self.ws
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    K = lay.K
    launches = 0
    data = [x.data_ptr()]  # the current buffer: x until the first reduction writes out

    def at(rr, off):
        return peer[rr] + off

    def wait(off, v):
        if v > 0:
            L.check(lib.gz_stream_wait_u32_geq(s, at(i, off), v), "gz_stream_wait_u32_geq")

    def signal(rr, off):
        L.check(lib.gz_stream_write_u32(s, at(rr, off), e), "gz_stream_write_u32")

    def msg(rr, k):  # (slots, sizes, widths) of the message rank rr sends as number k
        return tuple(at(rr, o) for o in lay.slot[k])

    def send(k, rr, src=None, k_in=None):
        """message k to rr: compress(data) or, with (src, k_in), the fused
        out = op(data, dec(src's message k_in)); compress(out)"""
        nonlocal launches
        wait(lay.consumed(k), prev)  # rr consumed our message k of the previous call
        io = _StepIO()
        io.out_slots, io.out_sizes, io.out_widths = msg(i, k)
        io.report_base = 0 if data[0] == x.data_ptr() else _NO_REPORT  # only x is the caller's input
        acc = None
        if src is not None:
            io.in_slots, io.in_sizes, io.in_widths = msg(src, k_in)
            acc = out.data_ptr()
        L.check(lib.gz_step(ctypes.byref(io), data[0], n, ebf, opc, acc, tws.data_ptr(), tws.numel(),
                            ws.status_ptr(), s), "gz_step")
        launches += 1
        data[0] = out.data_ptr() if acc is not None else data[0]
        signal(rr, lay.full(k))

    def receive_last(src, k_in, reduce: bool):  # out = [op(data,] dec(src's message k_in)[)]
        nonlocal launches
        io = _StepIO()
        io.in_slots, io.in_sizes, io.in_widths = msg(src, k_in)
        io.report_base = 0 if data[0] == x.data_ptr() else _NO_REPORT
        L.check(lib.gz_step_reduce(ctypes.byref(io), data[0] if reduce else None, n, ebf, opc, out.data_ptr(),
                                   ws.status_ptr(), s), "gz_step_reduce")
        launches += 1

    from .schedule import RdRecvLast, RdSend, rd_allreduce_plan

    for p in rd_allreduce_plan(N, i):  # the per-rank plan also run over gloo by the CPU tests
        if isinstance(p, RdSend):
            if p.src is not None:
                wait(lay.full(p.k_in), e)  # the sender posted its message k_in
            send(p.k, p.dst, src=p.src, k_in=p.k_in)
        else:
            wait(lay.full(p.k_in), e)
            receive_last(p.src, p.k_in, reduce=p.reduce)
        if p.src is not None:
            signal(p.src, lay.consumed(p.k_in))  # its message buffer is free again
    self._rd_epoch = e
    self.launches_per_call = launches
    if check:
        self.check()
    return out


def _rd_close(self):
    peers = getattr(self, "_rd_peer", None)
    if peers is not None:
        lib = L.lib()
        torch.cuda.synchronize(self.device)
        for r, p in enumerate(peers):
            if r != self.rank and p:
                lib.gz_ipc_close(p)
    self._rd_peer = None
    self._rd_buf = None
    self._rd_key = None


Communicator.rd_allreduce = rd_allreduce

from . import comm_generic as _comm_generic  # noqa: E402,F401  (comparator collectives, attached to Communicator)
