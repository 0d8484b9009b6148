"""The per-rank plans (schedule.py) executed by real processes over gloo on
the CPU, with the C oracle codec as the transport's compressor: every rank's
output must equal the reference's per-rank output bit for bit.  This covers
the N>1 schedule logic of the device path without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_data as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_PENDING = []


def _send_bytes(b: bytes, dst: int):
    """Non-blocking send (length, then payload); handles kept until the end."""
    n = torch.tensor([len(b)], dtype=torch.int64)
    _PENDING.append((n, dist.isend(n, dst)))
    if b:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        _PENDING.append((t, dist.isend(t, dst)))


def _recv_bytes(src: int) -> bytes:
    n = torch.empty(1, dtype=torch.int64)
    dist.recv(n, src)
    t = torch.empty(int(n.item()), dtype=torch.uint8)
    if t.numel():
        dist.recv(t, src)
    return t.numpy().tobytes()


def _worker(rank, world, port, case_idx, q):
    import sys

    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    from oracle import oracle as O
    from paper_2308_05199_b200.collectives import chunk_spans
    from paper_2308_05199_b200.schedule import Compress, Gather, Reduce, ring_allreduce_plan
    import golden_data as GG

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = GG.ring_cases()[case_idx]
    x = np.ascontiguousarray(case.inputs[rank], "<f4")
    N = world
    spans = chunk_spans(x.size, N)
    out = np.empty_like(x)
    right, left = (rank + 1) % N, (rank - 1) % N
    own_blob = None
    sent = []
    for p in ring_allreduce_plan(N, rank):
        if isinstance(p, Compress):
            lo, hi = spans[p.chunk]
            blob = O.compress(x[lo:hi], case.eb)
            sent.append(("rs", 0, blob))
            _send_bytes(blob, p.dst)
        elif isinstance(p, Reduce):
            blob = _recv_bytes(left)
            lo, hi = spans[p.chunk]
            acc = O.apply_op(case.op, x[lo:hi], O.decompress(blob))
            if p.last:
                out[lo:hi] = acc
                own_blob = O.compress(acc, case.eb)
            else:
                nb = O.compress(acc, case.eb)
                sent.append(("rs", p.slot + 1, nb))
                _send_bytes(nb, p.dst)
        elif isinstance(p, Gather):
            pass
    for _, h in _PENDING:
        h.wait()
    blobs = [None] * N
    dist.all_gather_object(blobs, own_blob)
    for p in ring_allreduce_plan(N, rank):
        if isinstance(p, Gather):
            lo, hi = spans[p.chunk]
            out[lo:hi] = O.decompress(blobs[p.owner])
    q.put((rank, out.tobytes(), [b for _, _, b in sent], own_blob))
    dist.barrier()
    dist.destroy_process_group()


CASES = [(k, c) for k, c in enumerate(G.ring_cases()) if c.algo == "ring-allreduce" and 2 <= c.N <= 8]


@pytest.mark.parametrize("k,case", CASES, ids=[f"N{c.N}-n{c.n}-{c.op}" for _, c in CASES])
def test_ring_allreduce_plan_over_gloo(k, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, case.N, port, k, q)) for r in range(case.N)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(case.N):
        r, out, sent, own = q.get(timeout=120)
        res[r] = (out, sent, own)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(case.N):
        assert res[r][0] == case.outputs[r].tobytes()
    # the RS messages each rank sent are the reference's traced RS messages
    N = case.N
    rs_msgs = case.msgs[: N * (N - 1)]
    for r in range(N):
        for s, blob in enumerate(res[r][1]):
            assert blob == rs_msgs[s * N + r]
        # the compress-once allgather blob is the reference's AG step-0 message
        assert res[r][2] == case.msgs[N * (N - 1) + r]
