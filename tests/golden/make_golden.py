"""Generate golden fixtures by running the REFERENCE gZCCL package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference is imported from ``baseline/_ref`` (installed from a copy of
/root/reference/pkg) or, failing that, from a scratch copy of
/root/reference/pkg/src.  Outputs (committed, small):

* ``blob_seed{1,2,3}.bin``  -- the reference's own golden cases
  (pkg/tests/conftest.py:7-13, pkg/tests/test_codec.py:183-189; those files
  were not shipped with the reference, this regenerates them).
* ``codec_cases.npz``       -- inputs / eb / blobs / block offsets for KATs,
  the reference's random byte-equality suite (test_codec.py:146-153) and
  edge cases (denormals, -0.0, huge/tiny eb, ties, raw blocks, partial blocks).
* ``ring_cases.npz``        -- ring-allreduce / reduce-scatter / allgather
  inputs, per-rank outputs and traced message payloads.
* ``scatter_cases.npz``     -- binomial-scatter inputs, outputs, messages.
* ``digests.json``          -- sha256 of large-field blobs (cfg1 at 3 eb).
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))


def import_reference():
    cand = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(cand, "gzccl")):
        sys.path.insert(0, cand)
    else:
        tmp = tempfile.mkdtemp(prefix="gzref_")
        shutil.copytree("/root/reference/pkg/src/gzccl", os.path.join(tmp, "gzccl"))
        sys.path.insert(0, tmp)
    import gzccl  # noqa: F401
    from gzccl import codec, collectives, simnet

    return codec, collectives, simnet


def pack_list(prefix, arrays, out):
    """Store a ragged list of 1-D arrays as one flat array + offsets."""
    lens = np.array([a.size for a in arrays], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    dt = arrays[0].dtype if arrays else np.uint8
    flat = np.concatenate(arrays).astype(dt) if arrays else np.empty(0, dt)
    out[prefix + "_flat"] = flat
    out[prefix + "_offs"] = offs


def smooth(n, phase=0.0):
    i = np.arange(n, dtype=np.float64)
    return (0.5 * np.sin(2 * np.pi * i / 65536 + phase) + 0.25 * np.sin(2 * np.pi * i / 4099 + phase)).astype(np.float32)


def codec_cases(codec):
    cases = []  # (name, x f32, eb)
    # conftest.py:7-13 golden cases
    for seed, (n, eb) in {1: (1000, 1e-3), 2: (4096, 1e-4), 3: (31, 1e-5)}.items():
        rng = np.random.default_rng(seed)
        cases.append((f"golden{seed}", rng.uniform(-1.0, 1.0, n).astype(np.float32), eb))
    # test_codec.py:55-84 KATs
    cases.append(("zeros1024", np.zeros(1024, np.float32), 1e-4))
    cases.append(("const314", np.full(1024, 3.14, np.float32), 1e-4))
    cases.append(("ramp1024", (np.arange(1024) * 0.001).astype(np.float32), 1e-4))
    cases.append(("zeros7", np.zeros(7, np.float32), 1e-3))
    cases.append(("empty", np.zeros(0, np.float32), 1e-4))
    # SURVEY §8(c) session KATs C1-C6
    cases.append(("C3ramp40", (np.arange(40) * 0.001).astype(np.float32), 1e-4))
    cases.append(("C4overflow", np.array([0, 1e30, 0], np.float32), 1e-4))
    cases.append(("C6tie", np.array([2.0**-53, 1.0], np.float32), 1.0))
    # test_codec.py:146-153 random suite (seed 77)
    rng = np.random.default_rng(77)
    for k in range(30):
        n = int(rng.integers(1, 200))
        scale = 10.0 ** float(rng.integers(-4, 8))
        data = (rng.uniform(-1, 1, n) * scale).astype(np.float32)
        eb = float(rng.choice([1e-3, 1e-4, 1e-6]))
        cases.append((f"rand77_{k}", data, eb))
    # test_codec.py:107-112 wild dynamic range
    rng = np.random.default_rng(5)
    data = (rng.uniform(-1, 1, 2000) * 10.0 ** rng.integers(-8, 25, 2000).astype(np.float64)).astype(np.float32)
    cases.append(("wild", data, 1e-5))
    # edge cases for the device kernels: every partial-block length, tiles
    rng = np.random.default_rng(2024)
    for n in (1, 2, 3, 31, 32, 33, 63, 64, 65, 255, 256, 257, 8191, 8192, 8193, 40000):
        cases.append((f"smooth_n{n}", smooth(n, 0.1 * n), 1e-4))
        cases.append((f"unif_n{n}", rng.uniform(0, 1, n).astype(np.float32), 1e-3))
    for eb in (1e-1, 1e-2, 1e-3, 1e-5, 1e-6, 1e-7, 3e-5, 0.5, 1.0, 2.0, 0.25, 1e3, 1e30, 1e-30, 1e-40, 1e-300, 1e300, 1e308,
               np.nextafter(0.5, 1.0), 5e-324, 1.7976931348623157e308):
        cases.append((f"eb_{eb!r}", np.concatenate([smooth(3000, 1.0) * 10, rng.normal(0, 1, 1000).astype(np.float32)]), float(eb)))
    tiny = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-40, -3e-39, 1.1754942e-38, 1.17549435e-38, 2e-38, -0.0, 0.0, 7e-46], np.float32)
    cases.append(("denormals_eb_tiny", np.tile(tiny, 20), 1e-44))
    cases.append(("denormals_eb_small", np.tile(tiny, 20), 1e-39))
    cases.append(("denormals_eb", np.tile(tiny, 20), 1e-4))
    big = np.array([3.4028235e38, -3.4028235e38, 3.4e38, 1e38, -1e38, 0.0, 3.4028235e38, 1.0], np.float32)
    for eb in (1e-4, 1e30, 1e37, 1e38, 3e38, 1e39, 1e100, 1e308):
        cases.append((f"big_eb_{eb!r}", np.tile(big, 9), float(eb)))
    ints = rng.integers(-100, 100, 5000).astype(np.float32)
    for eb in (0.5, 0.25, 1.0, 0.49999999999999994, 0.5000000000000001, 2.0**-20):
        cases.append((f"ints_eb_{eb!r}", ints, float(eb)))
    half = (np.arange(4000) * 0.5).astype(np.float32)  # exact ties of (x-prev)/tw
    for eb in (0.25, 0.125, 0.5, 1.0 / 3.0, 0.1):
        cases.append((f"halves_eb_{eb!r}", half, float(eb)))
    ramp_ties = (np.arange(3000, dtype=np.float64) * 3e-4).astype(np.float32)
    cases.append(("ramp_ties", ramp_ties, 1e-4))
    cases.append(("randwalk", np.cumsum(rng.normal(0, 1e-3, 20000)).astype(np.float32), 1e-4))
    cases.append(("randwalk_big", (1000 + np.cumsum(rng.normal(0, 1e-2, 20000))).astype(np.float32), 1e-4))
    cases.append(("step_w32", np.array([0, 3e5, -3e5, 3e5, -3e5] * 13, np.float32), 1e-4))
    for w in range(0, 33):
        # a block whose widest step needs exactly w bits (zigzag)
        step = 0 if w == 0 else (1 << (w - 1))
        x = np.zeros(64, np.float64)
        x[5] = step * 2e-3  # eb 1e-3 -> tw 2e-3
        cases.append((f"width{w}", x.astype(np.float32), 1e-3))
    names, xs, ebs, blobs, offs, ys = [], [], [], [], [], []
    for name, x, eb in cases:
        blob = codec.compress(x, eb)
        names.append(name)
        xs.append(np.ascontiguousarray(x, np.float32))
        ebs.append(eb)
        blobs.append(np.frombuffer(blob, np.uint8).copy())
        ys.append(np.asarray(codec.decompress(blob), np.float32))
        # block offsets as the reference computes them (codec.py:241-243) by
        # re-walking the payload exactly like decompress (codec.py:305-320)
        n = x.size
        nb = -(-n // 32)
        pos, o = 0, []
        payload = blob[24:]
        for i in range(nb):
            cnt = 32 if i < nb - 1 else n - (nb - 1) * 32
            w = payload[pos]
            o.append(pos)
            pos += 1 + 4 * cnt if w == 255 else 5 + ((cnt - 1) * w + 7) // 8
        assert pos == len(payload)
        offs.append(np.array(o, np.int64))
    out = {"names": np.array(names), "ebs": np.array(ebs, np.float64)}
    pack_list("x", xs, out)
    pack_list("blob", blobs, out)
    pack_list("boffs", offs, out)
    pack_list("y", ys, out)
    np.savez_compressed(os.path.join(HERE, "codec_cases.npz"), **out)
    return len(cases)


def ring_cases(codec, collectives, simnet):
    rows = []
    cfgs = [(2, 50, "sum", 1e-4), (3, 100, "sum", 1e-3), (4, 2, "sum", 1e-4), (4, 64, "max", 1e-4), (4, 1000, "sum", 1e-4),
            (5, 777, "sum", 1e-4), (8, 4099, "sum", 1e-4), (8, 5, "sum", 1e-4), (6, 3000, "max", 1e-3), (8, 20000, "sum", 1e-4),
            (2, 0, "sum", 1e-4), (1, 100, "sum", 1e-4), (7, 9000, "sum", 1e-5)]
    out = {}
    k = 0
    for algo in ("ring-allreduce", "ring-reduce-scatter", "ring-allgather"):
        for N, n, op, eb in cfgs:
            if algo != "ring-allreduce" and (n > 4099 or op == "max"):
                continue
            rng = np.random.default_rng(1000 + k)
            if algo == "ring-allgather":
                lens = [int(rng.integers(0, n + 1)) for _ in range(N)]
                inputs = [smooth(m, 0.37 * r) for r, m in enumerate(lens)]
            else:
                inputs = [smooth(n, 0.37 * r) + rng.normal(0, 1e-3, n).astype(np.float32) for r in range(N)]
            net = simnet.Network(simnet.CommunicatorSpec(N), record_payloads=True)
            outputs, rep = simnet.run_collective(net, algo, inputs, eb=eb, reduce_op=op, compute_accuracy=False)
            pre = f"c{k}_"
            out[pre + "meta"] = np.array([N, n, 1 if op == "max" else 0], np.int64)
            out[pre + "algo"] = np.array(algo)
            out[pre + "eb"] = np.array(eb)
            pack_list(pre + "in", [np.asarray(a, np.float32) for a in inputs], out)
            pack_list(pre + "out", [np.asarray(o, np.float32) for o in outputs], out)
            pack_list(pre + "msg", [np.frombuffer(t[3], np.uint8).copy() for t in net.trace], out)
            out[pre + "msg_src"] = np.array([t[0] for t in net.trace], np.int64)
            out[pre + "msg_dst"] = np.array([t[1] for t in net.trace], np.int64)
            rows.append((algo, N, n, op, eb))
            k += 1
    # recursive doubling (collectives.py:349-424), appended so earlier cases keep their seeds
    rd_cfgs = [(2, 100, "sum", 1e-4), (3, 257, "sum", 1e-4), (4, 1000, "sum", 1e-3), (5, 64, "max", 1e-4),
               (6, 3000, "sum", 1e-4), (7, 31, "sum", 1e-4), (8, 4099, "sum", 1e-4), (8, 700, "max", 1e-3),
               (4, 0, "sum", 1e-4), (1, 50, "sum", 1e-4), (3, 20000, "sum", 1e-5)]
    for N, n, op, eb in rd_cfgs:
        rng = np.random.default_rng(1000 + k)
        inputs = [smooth(n, 0.37 * r) + rng.normal(0, 1e-3, n).astype(np.float32) for r in range(N)]
        net = simnet.Network(simnet.CommunicatorSpec(N), record_payloads=True)
        outputs, rep = simnet.run_collective(net, "rd-allreduce", inputs, eb=eb, reduce_op=op, compute_accuracy=False)
        pre = f"c{k}_"
        out[pre + "meta"] = np.array([N, n, 1 if op == "max" else 0], np.int64)
        out[pre + "algo"] = np.array("rd-allreduce")
        out[pre + "eb"] = np.array(eb)
        pack_list(pre + "in", [np.asarray(a, np.float32) for a in inputs], out)
        pack_list(pre + "out", [np.asarray(o, np.float32) for o in outputs], out)
        pack_list(pre + "msg", [np.frombuffer(t[3], np.uint8).copy() for t in net.trace], out)
        out[pre + "msg_src"] = np.array([t[0] for t in net.trace], np.int64)
        out[pre + "msg_dst"] = np.array([t[1] for t in net.trace], np.int64)
        rows.append(("rd-allreduce", N, n, op, eb))
        k += 1
    # comparators (collectives.py:311-341, 545-566): the compress-per-hop allgather and the lossless twins
    cmp_cfgs = [("cprp2p-allgather", 2, 300, "sum", 1e-4), ("cprp2p-allgather", 4, 1000, "sum", 1e-3),
                ("cprp2p-allgather", 7, 64, "sum", 1e-4), ("lossless-allreduce", 4, 1000, "sum", 1e-4),
                ("lossless-allreduce", 3, 77, "max", 1e-4), ("lossless-reduce-scatter", 5, 999, "sum", 1e-4),
                ("lossless-allgather", 4, 500, "sum", 1e-4)]
    for algo, N, n, op, eb in cmp_cfgs:
        rng = np.random.default_rng(1000 + k)
        if algo.endswith("allgather"):
            lens = [int(rng.integers(0, n + 1)) for _ in range(N)]
            inputs = [smooth(m, 0.37 * r) for r, m in enumerate(lens)]
        else:
            inputs = [smooth(n, 0.37 * r) + rng.normal(0, 1e-3, n).astype(np.float32) for r in range(N)]
        net = simnet.Network(simnet.CommunicatorSpec(N), record_payloads=True)
        outputs, rep = simnet.run_collective(net, algo, inputs, eb=eb, reduce_op=op, compute_accuracy=False)
        pre = f"c{k}_"
        out[pre + "meta"] = np.array([N, n, 1 if op == "max" else 0], np.int64)
        out[pre + "algo"] = np.array(algo)
        out[pre + "eb"] = np.array(eb)
        pack_list(pre + "in", [np.asarray(a, np.float32) for a in inputs], out)
        pack_list(pre + "out", [np.asarray(o, np.float32) for o in outputs], out)
        pack_list(pre + "msg", [np.frombuffer(t[3], np.uint8).copy() for t in net.trace], out)
        out[pre + "msg_src"] = np.array([t[0] for t in net.trace], np.int64)
        out[pre + "msg_dst"] = np.array([t[1] for t in net.trace], np.int64)
        rows.append((algo, N, n, op, eb))
        k += 1
    out["count"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "ring_cases.npz"), **out)
    return rows


def scatter_cases(codec, collectives, simnet):
    cfgs = [(2, [500, 500], 0), (3, None, 0), (4, [1, 1, 1, 1], 0), (4, [3, 4, 5, 2], 2), (6, [7, 3, 9, 2, 5, 4], 0),
            (8, None, 0), (8, [0, 100, 0, 5000, 1, 2, 33, 4000], 5), (5, [0, 0, 0, 0, 0], 1), (1, None, 0), (7, None, 3),
            (16, None, 0)]
    out = {}
    for k, (N, counts, root) in enumerate(cfgs):
        total = sum(counts) if counts is not None else 10000 + 37 * N
        data = smooth(total, 0.5) + np.random.default_rng(k).normal(0, 1e-3, total).astype(np.float32)
        net = simnet.Network(simnet.CommunicatorSpec(N, root=root), record_payloads=True)
        outputs, _ = simnet.run_collective(net, "binomial-scatter", data, eb=1e-4, counts=counts, compute_accuracy=False)
        pre = f"s{k}_"
        out[pre + "meta"] = np.array([N, root], np.int64)
        out[pre + "counts"] = np.array(counts if counts is not None else [], np.int64)
        out[pre + "data"] = data
        pack_list(pre + "out", [np.asarray(o, np.float32) for o in outputs], out)
        pack_list(pre + "msg", [np.frombuffer(t[3], np.uint8).copy() for t in net.trace], out)
        out[pre + "msg_src"] = np.array([t[0] for t in net.trace], np.int64)
        out[pre + "msg_dst"] = np.array([t[1] for t in net.trace], np.int64)
    out["count"] = np.array(len(cfgs))
    np.savez_compressed(os.path.join(HERE, "scatter_cases.npz"), **out)
    return len(cfgs)


def fixed_rate_cases(codec):
    """Fixed-rate baseline codec (codec.py:442-489): inputs, bits, blobs, decoded values."""
    cfgs = [(0, 8), (1, 4), (31, 1), (32, 3), (1000, 8), (4099, 16), (777, 5), (20000, 12), (64, 7), (100, 2)]
    out = {}
    datas, blobs, ys = [], [], []
    for k, (n, b) in enumerate(cfgs):
        rng = np.random.default_rng(2000 + k)
        x = smooth(n, 0.2 * k) + rng.normal(0, 0.01, n).astype(np.float32) if k % 3 else rng.uniform(-5, 5, n).astype(np.float32)
        if k == 9:
            x = np.full(n, 3.25, np.float32)  # hi == lo
        blob = codec.fixed_rate_compress(x, b)
        datas.append(np.asarray(x, np.float32))
        blobs.append(np.frombuffer(blob, np.uint8).copy())
        ys.append(codec.fixed_rate_decompress(blob))
    out["bits"] = np.array([b for _, b in cfgs], np.int64)
    pack_list("x", datas, out)
    pack_list("blob", blobs, out)
    pack_list("y", ys, out)
    out["count"] = np.array(len(cfgs))
    np.savez_compressed(os.path.join(HERE, "fixed_rate_cases.npz"), **out)
    return len(cfgs)


def fixed_rate_zero_cases(codec):
    """Fixed-rate blobs whose min and/or max is a zero: the header carries the
    sign numpy's SIMD reduction returns (order-dependent for +-0).  Generated on
    an AVX-512 host (numpy dispatch AVX512_SKX); other hosts' numpy may differ,
    which is why the oracle restates the AVX-512 reduction explicitly."""
    from numpy._core._multiarray_umath import __cpu_features__ as feats

    assert feats.get("AVX512_SKX"), "generate these on an AVX-512 host"
    rng = np.random.default_rng(4242)
    datas, blobs, ys, bits = [], [], [], []
    lengths = [1, 2, 3, 16, 17, 18, 31, 33, 64, 129, 130, 257, 1000, 4097, 20001]
    for k, n in enumerate(lengths * 2):
        x = np.zeros(n, np.float32)
        kind = k % 4
        if kind == 1:
            x = rng.integers(0, 3, n).astype(np.float32)     # min is a zero
        elif kind == 2:
            x = -rng.integers(0, 3, n).astype(np.float32)    # max is a zero
        elif kind == 3:
            x = rng.uniform(-1, 1, n).astype(np.float32)
            x[rng.random(n) < 0.3] = 0.0                    # zeros inside, extremum not zero
        z = x == 0
        x[z] = np.where(rng.random(int(z.sum())) < rng.random(), -0.0, 0.0).astype(np.float32)
        b = int(1 + k % 16)
        blob = codec.fixed_rate_compress(x, b)
        datas.append(x)
        blobs.append(np.frombuffer(blob, np.uint8).copy())
        ys.append(codec.fixed_rate_decompress(blob))
        bits.append(b)
    out = {"bits": np.array(bits, np.int64), "count": np.array(len(bits))}
    pack_list("x", datas, out)
    pack_list("blob", blobs, out)
    pack_list("y", ys, out)
    np.savez_compressed(os.path.join(HERE, "fixed_rate_zero_cases.npz"), **out)
    return len(bits)


def digests(codec):
    x = smooth(1 << 24)
    d = {"cfg1_input_sha256": hashlib.sha256(x.tobytes()).hexdigest()}
    for eb in (1e-4, 1e-3, 1e-2):
        blob = codec.compress(x, eb)
        d[f"cfg1_eb{eb!r}"] = {"len": len(blob), "sha256": hashlib.sha256(blob).hexdigest()}
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(d, f, indent=1)
    return d


if __name__ == "__main__":
    codec, collectives, simnet = import_reference()
    for seed, (n, eb) in {1: (1000, 1e-3), 2: (4096, 1e-4), 3: (31, 1e-5)}.items():
        rng = np.random.default_rng(seed)
        data = rng.uniform(-1.0, 1.0, n).astype(np.float32)
        with open(os.path.join(HERE, f"blob_seed{seed}.bin"), "wb") as f:
            f.write(codec.compress(data, eb))
    print("codec cases:", codec_cases(codec))
    print("ring cases:", len(ring_cases(codec, collectives, simnet)))
    print("fixed-rate cases:", fixed_rate_cases(codec))
    print("fixed-rate signed-zero cases:", fixed_rate_zero_cases(codec))
    print("scatter cases:", scatter_cases(codec, collectives, simnet))
    print("digests:", digests(codec))
