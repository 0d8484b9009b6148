"""Multi-GPU parity worker (launched by tests/test_comm_gpu.py via torchrun).

Each rank runs Communicator.ring_allreduce on its own GPU (NVLink peer memory)
and compares its output byte-for-byte with the CPU oracle's per-rank output
for the same inputs (and with the reference's golden per-rank outputs for the
golden cases of matching rank count).
"""

import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # rehearsal of rank counts above the box's GPU count (tools/gpu_n8_rehearsal.sh):
    # several ranks share a GPU, so NCCL (one rank per GPU) is replaced by gloo for
    # the object plumbing; the data path is the same CUDA-IPC peer memory
    oversub = world > torch.cuda.device_count()
    local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    from oracle import oracle as O
    from paper_2308_05199_b200 import comm
    import golden_data as G

    c = comm.Communicator(dist.group.WORLD, dev)
    failures = []
    checked = 0
    # golden cases (reference outputs) with this rank count
    for case in G.ring_cases():
        if case.algo != "ring-allreduce" or case.N != world:
            continue
        x = torch.from_numpy(np.ascontiguousarray(case.inputs[rank], np.float32)).to(dev)
        for rep in range(2):  # twice: flags and slots are reused across calls
            out = c.ring_allreduce(x, case.eb, case.op)
            torch.cuda.synchronize()
            if out.cpu().numpy().tobytes() != case.outputs[rank].tobytes():
                failures.append(f"golden N={case.N} n={case.n} op={case.op} rep={rep}")
            checked += 1
    # larger seeded inputs vs the oracle
    rng = np.random.default_rng(7)
    for n, op, eb in ((1 << 20, "sum", 1e-4), (3_000_017, "sum", 1e-3), (777_777, "max", 1e-4), (1 << 22, "sum", 1e-5)):
        bufs = [O.smooth_field(n, 0.37 * r) + np.random.default_rng(100 + r).normal(0, 1e-3, n).astype(np.float32)
                for r in range(world)]
        expect = O.ring_allreduce(bufs, eb, op)
        x = torch.from_numpy(bufs[rank]).to(dev)
        for mode in ("slots", "copy", "multi", "auto"):  # the allgather's data paths
            c.ag_mode = mode
            c.kernel_waits = mode != "copy"  # ring flags taken by stream wait nodes or inside the kernels
            out = c.ring_allreduce(x, eb, op)
            torch.cuda.synchronize()
            if out.cpu().numpy().tobytes() != expect[rank].tobytes():
                failures.append(f"oracle n={n} op={op} eb={eb} ag_mode={mode}")
            checked += 1
    c.ag_mode = "slots"
    c.kernel_waits = True
    # repeated calls on the same tensors are replayed from a captured CUDA graph
    n = 3_000_017
    bufs = [O.smooth_field(n, 0.21 * r) + np.random.default_rng(900 + r).normal(0, 1e-3, n).astype(np.float32)
            for r in range(world)]
    expect = O.ring_allreduce(bufs, 1e-4, "sum")[rank].tobytes()
    expect0 = expect
    expect1 = O.ring_allreduce([bufs[(r + 1) % world] for r in range(world)], 1e-4, "sum")[rank].tobytes()
    for mode in ("slots", "copy", "multi"):
        c.ag_mode = mode
        x = torch.from_numpy(bufs[rank]).to(dev)
        out = torch.empty_like(x)
        expect = expect0
        for rep in range(5):
            if rep == 3:
                x.copy_(torch.from_numpy(bufs[(rank + 1) % world]))  # new values, same tensors: the graph sees them
                expect = expect1
            c.ring_allreduce(x, 1e-4, "sum", out=out)
            torch.cuda.synchronize()
            if out.cpu().numpy().tobytes() != expect:
                failures.append(f"graph replay rep={rep} ag_mode={mode}")
            checked += 1
    c.ag_mode = "slots"
    if not c._graph_cache:
        failures.append("no graph was captured")
    # standalone reduce-scatter and allgather(v) (collectives.py:247-291), vs the oracle,
    # interleaved with allreduce calls (shared flags and slots)
    for n, op, eb in ((1 << 20, "sum", 1e-4), (999_999, "max", 1e-3), (5, "sum", 1e-4)):
        bufs = [O.smooth_field(n, 0.29 * r) + np.random.default_rng(300 + r).normal(0, 1e-3, n).astype(np.float32)
                for r in range(world)]
        expect = O.ring_reduce_scatter(bufs, eb, op)
        got = c.ring_reduce_scatter(torch.from_numpy(bufs[rank]).to(dev), eb, op)
        torch.cuda.synchronize()
        if got.cpu().numpy().tobytes() != np.ascontiguousarray(expect[rank], np.float32).tobytes():
            failures.append(f"reduce_scatter n={n} op={op}")
        checked += 1
        out = c.ring_allreduce(torch.from_numpy(bufs[rank]).to(dev), eb, op)
        torch.cuda.synchronize()
        if out.cpu().numpy().tobytes() != O.ring_allreduce(bufs, eb, op)[rank].tobytes():
            failures.append(f"allreduce after reduce_scatter n={n}")
        checked += 1
    for sizes in ([1 << 18] * world, [1000 + 77 * r for r in range(world)], [0] + [4096] * (world - 1)):
        chunks = [O.smooth_field(sz, 0.5 * r) for r, sz in enumerate(sizes)]
        expect = O.ring_allgather(chunks, 1e-4)
        for rep in range(2):
            got = c.ring_allgather(torch.from_numpy(chunks[rank]).to(dev), 1e-4)
            torch.cuda.synchronize()
            if got.cpu().numpy().tobytes() != np.ascontiguousarray(expect[rank], np.float32).tobytes():
                failures.append(f"allgather sizes={sizes[:3]} rep={rep}")
            checked += 1
    # recursive-doubling allreduce (collectives.py:349-424): golden cases, then the oracle
    for case in G.ring_cases():
        if case.algo != "rd-allreduce" or case.N != world:
            continue
        for rep in range(2):
            got = c.rd_allreduce(torch.from_numpy(np.ascontiguousarray(case.inputs[rank], np.float32)).to(dev), case.eb,
                                 case.op)
            torch.cuda.synchronize()
            if got.cpu().numpy().tobytes() != case.outputs[rank].tobytes():
                failures.append(f"rd golden N={case.N} n={case.n} op={case.op} rep={rep}")
            checked += 1
    for n, op, eb in ((1 << 20, "sum", 1e-4), (333_333, "max", 1e-3), (1 << 22, "sum", 1e-5)):
        bufs = [O.smooth_field(n, 0.41 * r) + np.random.default_rng(500 + r).normal(0, 1e-3, n).astype(np.float32)
                for r in range(world)]
        expect = O.rd_allreduce(bufs, eb, op)
        got = c.rd_allreduce(torch.from_numpy(bufs[rank]).to(dev), eb, op)
        torch.cuda.synchronize()
        if got.cpu().numpy().tobytes() != expect[rank].tobytes():
            failures.append(f"rd oracle n={n} op={op}")
        checked += 1
    # binomial scatter: golden cases of this rank count, then seeded cases at every root
    for case in G.scatter_cases():
        if case.N != world:
            continue
        for routing in ("tree", "direct"):
            for rep in range(2):
                x = torch.from_numpy(np.ascontiguousarray(case.data, np.float32)).to(dev) if rank == case.root else None
                out = c.binomial_scatter(x, 1e-4, counts=case.counts, root=case.root, routing=routing)
                torch.cuda.synchronize()
                if out.cpu().numpy().tobytes() != case.outputs[rank].tobytes():
                    failures.append(f"scatter golden root={case.root} counts={case.counts} {routing} rep={rep}")
                checked += 1
    for n, eb, counts in ((1 << 22, 1e-4, None), (1_000_003, 1e-3, None),
                          (9_999, 1e-4, [0] * (world - 1) + [9_999]),
                          (5_000_000, 1e-5, [5_000_000 // world + (7 if r % 2 else -7) for r in range(world)])):
        data = O.smooth_field(n, 0.11) + np.random.default_rng(n).normal(0, 1e-3, n).astype(np.float32)
        if counts is not None and sum(counts) != n:
            counts[-1] += n - sum(counts)
        for root in range(world):
            expect = O.binomial_scatter(data, world, eb, root=root, counts=counts)
            for routing in ("tree", "direct"):
                x = torch.from_numpy(data).to(dev) if rank == root else None
                out = c.binomial_scatter(x, eb, counts=counts, root=root, routing=routing)
                torch.cuda.synchronize()
                if out.cpu().numpy().tobytes() != expect[rank].tobytes():
                    failures.append(f"scatter oracle n={n} eb={eb} root={root} {routing}")
                checked += 1
    # bad counts: every rank raises the root's error
    try:
        c.binomial_scatter(torch.zeros(10, device=dev) if rank == 0 else None, 1e-4, counts=[1] * world, root=0)
        failures.append("bad counts accepted")
    except ValueError as err:
        if "sum" not in str(err):
            failures.append(f"bad counts message {err}")
    checked += 1
    # a captured ring graph must survive other collectives growing the communicator's
    # workspace (the ring has its own, sized once per setup)
    n = 1 << 20
    bufs = [O.smooth_field(n, 0.13 * r) for r in range(world)]
    expect = O.ring_allreduce(bufs, 1e-4, "sum")[rank].tobytes()
    x = torch.from_numpy(bufs[rank]).to(dev)
    out = torch.empty_like(x)
    for rep in range(3):
        c.ring_allreduce(x, 1e-4, "sum", out=out)
    big = [O.smooth_field(6_000_000, 0.3 * r) for r in range(world)]
    c.rd_allreduce(torch.from_numpy(big[rank]).to(dev), 1e-4)  # grows the shared tile workspace
    if rank == 0:
        xb = torch.from_numpy(O.smooth_field(8_000_000, 0.2)).to(dev)
    c.binomial_scatter(xb if rank == 0 else None, 1e-4, root=0)
    for rep in range(2):
        c.ring_allreduce(x, 1e-4, "sum", out=out)  # graph replay
        torch.cuda.synchronize()
        if out.cpu().numpy().tobytes() != expect:
            failures.append(f"ring graph replay after workspace growth rep={rep}")
        checked += 1
    # errors (codec.py:79-86 via collectives.py:202-205): a non-finite input value raises on
    # EVERY rank with the offset of the first bad value in rank order; the communicator
    # stays usable afterwards
    def expect_error(what, fn, frag):
        nonlocal checked
        try:
            fn()
            failures.append(f"{what}: no error raised")
        except ValueError as err:
            if frag not in str(err):
                failures.append(f"{what}: message {err!r}, expected {frag!r}")
        checked += 1
    n = 100_003
    for bad_rank, off in ((1, 54_321), (world - 1, 7)):
        for kind in ("allreduce", "reduce_scatter", "rd"):
            xs = [O.smooth_field(n, 0.5 * r) for r in range(world)]
            xs[bad_rank][off] = np.nan
            if world > 2 and bad_rank == 1:
                xs[2][3] = np.inf  # later in rank order: the rank-1 offset is reported
            xt = torch.from_numpy(xs[rank]).to(dev)
            fn = {"allreduce": lambda: c.ring_allreduce(xt, 1e-4),
                  "reduce_scatter": lambda: c.ring_reduce_scatter(xt, 1e-4),
                  "rd": lambda: c.rd_allreduce(xt, 1e-4)}[kind]
            expect_error(f"{kind} nan rank={bad_rank} off={off}", fn, f"non-finite value at offset {off}")
    for root, off in ((0, 3), (0, n - 1), (world - 1, 3), (world - 1, n - 1)):  # own block / a sent block
        data = O.smooth_field(n, 0.9)
        data[off] = -np.inf
        xt = torch.from_numpy(data).to(dev) if rank == root else None
        expect_error(f"scatter inf root={root} off={off}", lambda: c.binomial_scatter(xt, 1e-4, root=root),
                     f"non-finite value at offset {off}")
    xs = [O.smooth_field(n, 0.5 * r) for r in range(world)]
    got = c.ring_allreduce(torch.from_numpy(xs[rank]).to(dev), 1e-4)
    torch.cuda.synchronize()
    if got.cpu().numpy().tobytes() != O.ring_allreduce(xs, 1e-4)[rank].tobytes():
        failures.append("allreduce after errors")
    checked += 1
    # the comparators on the real multi-GPU path (collectives.py:94-194, 311-341): lossless twins,
    # the fixed-rate transport and the compress-per-hop allgather, vs the single-GPU schedules
    # (themselves bit-exact vs the reference, tests/test_transport_gpu.py) and the reference goldens
    from paper_2308_05199_b200 import collectives as C
    for case in G.ring_cases():
        if case.N != world or case.algo not in ("lossless-allreduce", "lossless-reduce-scatter",
                                                "lossless-allgather", "cprp2p-allgather"):
            continue
        xin = torch.from_numpy(np.ascontiguousarray(case.inputs[rank], np.float32)).to(dev)
        for rep in range(2):
            if case.algo == "lossless-allreduce":
                got = c.lossless_allreduce(xin, case.op)
            elif case.algo == "lossless-reduce-scatter":
                got = c.lossless_reduce_scatter(xin, case.op)
            elif case.algo == "lossless-allgather":
                got = c.lossless_allgather(xin)
            else:
                got = c.cprp2p_allgather(xin, case.eb)
            if got.cpu().numpy().tobytes() != np.ascontiguousarray(case.outputs[rank], np.float32).tobytes():
                failures.append(f"{case.algo} golden N={case.N} rep={rep}")
            checked += 1
    for n, op in ((300_007, "sum"), (65_536, "max")):
        bufs = [O.smooth_field(n, 0.23 * r) + np.random.default_rng(700 + r).normal(0, 1e-2, n).astype(np.float32)
                for r in range(world)]
        xin = torch.from_numpy(bufs[rank]).to(dev)
        for algo, codec, fn in (("lossless-allreduce", "ebz", lambda: c.lossless_allreduce(xin, op)),
                                ("ring-allreduce", "fixed-rate", lambda: c.fixed_rate_allreduce(xin, 9, op)),
                                ("lossless-reduce-scatter", "ebz", lambda: c.lossless_reduce_scatter(xin, op)),
                                ("ring-reduce-scatter", "fixed-rate",
                                 lambda: c.generic_reduce_scatter(xin, "fixed-rate", bits=9, op=op)),
                                ("ring-allgather", "fixed-rate", lambda: c.generic_allgather(xin, "fixed-rate", bits=9)),
                                ("cprp2p-allgather", "ebz", lambda: c.cprp2p_allgather(xin, 1e-3))):
            ref_out, _ = C.run_collective(world, algo, bufs, eb=1e-3, codec=codec, bits=9, reduce_op=op,
                                          compute_accuracy=False)
            for rep in range(2):
                got = fn()
                if got.cpu().numpy().tobytes() != np.ascontiguousarray(ref_out[rank], np.float32).tobytes():
                    failures.append(f"{algo}/{codec} n={n} op={op} rep={rep}")
                checked += 1
    flag = torch.tensor([len(failures)], device="cpu" if oversub else dev)
    dist.all_reduce(flag)
    if rank == 0:
        print(f"mgpu ranks={world} checked={checked} failures={int(flag.item())}", flush=True)
    if failures:
        print(f"rank {rank} failures: {failures}", flush=True)
    c.close()
    dist.destroy_process_group()
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
