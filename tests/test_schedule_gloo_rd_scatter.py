"""The recursive-doubling plan (schedule.rd_allreduce_plan, the one comm.py
executes) and the binomial-scatter tree (schedule.scatter_route) run by real
processes over gloo on the CPU, the C oracle as the codec: every rank's output
and every message must equal the reference's (golden fixtures made by running
gzccl: collectives.py:349-424 rd_allreduce_c, 467-532 binomial_scatter_c).
This covers the donor / absorber roles and the tree's byte-range forwarding
without a GPU."""

import os
import socket
import struct

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_data as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys

    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


class _Wire:
    """Length-prefixed byte messages over gloo point-to-point (simnet.py:119-137)."""

    def __init__(self):
        import torch

        self.torch = torch
        self.pending = []

    def send(self, b: bytes, dst: int):
        torch = self.torch
        n = torch.tensor([len(b)], dtype=torch.int64)
        self.pending.append((n, dist.isend(n, dst)))
        if b:
            t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
            self.pending.append((t, dist.isend(t, dst)))

    def recv(self, src: int) -> bytes:
        torch = self.torch
        n = torch.empty(1, dtype=torch.int64)
        dist.recv(n, src)
        t = torch.empty(int(n.item()), dtype=torch.uint8)
        if t.numel():
            dist.recv(t, src)
        return t.numpy().tobytes()

    def drain(self):
        for _, h in self.pending:
            h.wait()


def _rd_case(rank, world, case_idx):
    from oracle import oracle as O
    from paper_2308_05199_b200.schedule import RdSend, rd_allreduce_plan
    import golden_data as GG

    case = GG.ring_cases()[case_idx]
    data = np.ascontiguousarray(case.inputs[rank], "<f4").copy()
    w = _Wire()
    sent = []
    for p in rd_allreduce_plan(world, rank):
        if p.src is not None:
            recv = O.decompress(w.recv(p.src))
            data = O.apply_op(case.op, data, recv) if (isinstance(p, RdSend) or p.reduce) else recv
        if isinstance(p, RdSend):
            blob = O.compress(data, case.eb)
            sent.append((rank, p.dst, blob))
            w.send(blob, p.dst)
    w.drain()
    return np.ascontiguousarray(data, "<f4").tobytes(), sent


RD = [(k, c) for k, c in enumerate(G.ring_cases()) if c.algo == "rd-allreduce" and c.N >= 2]


@pytest.mark.parametrize("k,case", RD, ids=[f"N{c.N}-n{c.n}-{c.op}" for _, c in RD])
def test_rd_allreduce_plan_over_gloo(k, case):
    res = _results(case.N)[("rd", k)]
    for r in range(case.N):
        assert res[r][0] == case.outputs[r].tobytes(), f"rank {r}"
    # every message the plan sends is one the reference sent (same src, dst, bytes)
    got = sorted((s, d, b) for r in range(case.N) for s, d, b in res[r][1])
    ref = sorted(zip((int(v) for v in case.src), (int(v) for v in case.dst), case.msgs))
    assert got == ref


def _scatter_case(rank, world, case_idx):
    from oracle import oracle as O
    from paper_2308_05199_b200.schedule import scatter_route
    import golden_data as GG

    case = GG.scatter_cases()[case_idx]
    N, root = world, case.root
    counts = case.counts or [hi - lo for lo, hi in O.chunk_spans(case.data.size, N)]
    parent, vr, sends = scatter_route(N, root)[rank]
    order = [(root + j) % N for j in range(N)]
    w = _Wire()
    sent = []
    hdr = struct.Struct("<QQQ")
    if rank == root:
        lo_ = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        blobs = [O.compress(case.data[lo_[r]:lo_[r + 1]], 1e-4) for r in order]  # virtual-rank order
        sizes = [len(b) for b in blobs]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
        payload = b"".join(blobs)
        base = 0
        out = np.ascontiguousarray(case.data[lo_[root]:lo_[root + 1]], "<f4")
    else:
        msg = w.recv(parent)
        cnt, lo, hi = hdr.unpack_from(msg)
        sizes = list(np.frombuffer(msg, "<u8", cnt, hdr.size).astype(int))
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
        payload = msg[hdr.size + 8 * cnt:]
        base = offs[lo]  # the fragment starts at block lo
        out = O.decompress(payload[offs[vr] - base:offs[vr] + sizes[vr] - base])
    for child, clo, chi in sends:  # forward the children's byte ranges unchanged
        frag = payload[offs[clo] - base:offs[chi - 1] + sizes[chi - 1] - base]
        m = hdr.pack(N, clo, chi) + np.asarray(sizes, "<u8").tobytes() + frag
        sent.append((rank, child, m))
        w.send(m, child)
    w.drain()
    return np.ascontiguousarray(out, "<f4").tobytes(), sent


SC = [(k, c) for k, c in enumerate(G.scatter_cases()) if c.N >= 2]


@pytest.mark.parametrize("k,case", SC, ids=[f"N{c.N}-root{c.root}" for _, c in SC])
def test_binomial_scatter_tree_over_gloo(k, case):
    res = _results(case.N)[("scatter", k)]
    for r in range(case.N):
        assert res[r][0] == case.outputs[r].tobytes(), f"rank {r}"
    got = sorted((s, d, b) for r in range(case.N) for s, d, b in res[r][1])
    ref = sorted(zip((int(v) for v in case.src), (int(v) for v in case.dst), case.msgs))
    assert got == ref


def _worker(rank, world, port, jobs, q):
    # one process group per rank count runs every case of that count in turn
    _init(rank, world, port)
    for kind, k in jobs:
        fn = _rd_case if kind == "rd" else _scatter_case
        out, sent = fn(rank, world, k)
        q.put((kind, k, rank, out, sent))
        dist.barrier()
    dist.destroy_process_group()


_CACHE = {}


def _results(N):
    if N not in _CACHE:
        jobs = [("rd", k) for k, c in RD if c.N == N] + [("scatter", k) for k, c in SC if c.N == N]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, N, port, jobs, q)) for r in range(N)]
        for p in procs:
            p.start()
        res = {}
        for _ in range(N * len(jobs)):
            kind, k, r, out, sent = q.get(timeout=300)
            res.setdefault((kind, k), {})[r] = (out, sent)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        _CACHE[N] = res
    return _CACHE[N]
