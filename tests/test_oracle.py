"""The CPU oracle (oracle/) is pinned against golden vectors produced by the
reference itself.  CPU-only."""

import hashlib

import numpy as np
import pytest

import golden_data as G
from conftest import max_err

CASES = G.codec_cases()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_oracle_compress_matches_reference(case, oracle):
    blob, offs = oracle.compress(case.x, case.eb, return_offsets=True)
    assert blob == case.blob
    if case.x.size:
        assert np.array_equal(offs, case.block_offsets)


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_oracle_decompress_matches_reference(case, oracle):
    y = oracle.decompress(case.blob)
    assert y.tobytes() == case.y.tobytes()


@pytest.mark.parametrize("threads", [2, 3, 8])
def test_oracle_threads_bit_identical(threads, oracle):
    for case in CASES[:60]:
        assert oracle.compress(case.x, case.eb, threads=threads) == case.blob
        assert oracle.decompress(case.blob, threads=threads).tobytes() == case.y.tobytes()


@pytest.mark.parametrize("seed", sorted(G.GOLDEN_CASES))
def test_oracle_golden_files(seed, oracle):
    data, eb = G.golden_data(seed)
    expected = G.golden_blob(seed)
    assert oracle.compress(data, eb) == expected
    assert max_err(data, oracle.decompress(expected)) <= eb


def test_oracle_session_kats(oracle):
    # SURVEY §8(c) C1, C2, C3, C4, C6
    assert oracle.compress(np.zeros(7, np.float32), 1e-3).hex() == "475a4331000000000700000000000000fca9f1d24d62503f0000000000"
    assert oracle.compress(np.zeros(3, np.float32), 1e-4)[:24].hex() == "475a43310000000003000000000000002d431cebe2361a3f"
    c3 = oracle.compress((np.arange(40) * 0.001).astype(np.float32), 1e-4)[24:]
    assert c3.hex() == "04" + "00000000" + "aa" * 15 + "0a" + "04" + "6f12033d" + "aaaaaa0a"
    assert oracle.compress(np.array([0, 1e30, 0], np.float32), 1e-4)[24:].hex() == "ff" + "00000000" + "caf24971" + "00000000"
    assert oracle.compress(np.array([2.0**-53, 1.0], np.float32), 1.0)[24:].hex() == "02" + "00000025" + "02"


def test_oracle_kat_sizes(oracle):
    # pkg/tests/test_codec.py:56-84
    assert len(oracle.compress(np.zeros(1024, np.float32), 1e-4)) == 184
    assert len(oracle.compress(np.full(1024, 3.14, np.float32), 1e-4)) == 24 + 32 * 5
    assert len(oracle.compress((np.arange(1024) * 0.001).astype(np.float32), 1e-4)) == 24 + 32 * 21
    assert len(oracle.compress(np.empty(0, np.float32), 1e-4)) == 24


def test_oracle_errors(oracle):
    with pytest.raises(ValueError, match="offset 2"):
        oracle.compress(np.array([0.0, 1.0, np.nan], np.float32), 1e-4)
    for eb in (0.0, -1e-4, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            oracle.compress(np.ones(4, np.float32), eb)
    blob = oracle.compress(np.zeros(64, np.float32), 1e-4)
    with pytest.raises(ValueError, match="trailing"):
        oracle.decompress(blob + b"\x00")
    bad = bytearray(blob)
    bad[24] = 77
    with pytest.raises(ValueError, match="width"):
        oracle.decompress(bytes(bad))
    with pytest.raises(ValueError, match="magic"):
        oracle.decompress(b"XXXX" + blob[4:])


def test_oracle_cfg1_digest(oracle):
    d = G.digests()
    x = oracle.smooth_field(1 << 24)
    if hashlib.sha256(x.tobytes()).hexdigest() != d["cfg1_input_sha256"]:
        pytest.skip("numpy sin differs on this host; cfg1 input not reproducible")
    blob = oracle.compress(x, 1e-4, threads=8)
    assert len(blob) == d["cfg1_eb0.0001"]["len"]
    assert hashlib.sha256(blob).hexdigest() == d["cfg1_eb0.0001"]["sha256"]


RING = G.ring_cases()


@pytest.mark.parametrize("case", RING, ids=[f"{c.algo}-N{c.N}-n{c.n}-{c.op}" for c in RING])
def test_oracle_ring_matches_reference(case, oracle):
    trace = []
    if case.algo == "ring-allreduce":
        outs = oracle.ring_allreduce(case.inputs, case.eb, case.op, trace)
    elif case.algo == "ring-reduce-scatter":
        outs = oracle.ring_reduce_scatter(case.inputs, case.eb, case.op, trace)
    elif case.algo == "rd-allreduce":
        outs = oracle.rd_allreduce(case.inputs, case.eb, case.op, trace)
    elif case.algo == "cprp2p-allgather":
        outs = oracle.cprp2p_allgather(case.inputs, case.eb, trace)
    elif case.algo == "lossless-allreduce":
        outs = oracle.ring_allreduce(case.inputs, case.eb, case.op, trace, raw=True)
    elif case.algo == "lossless-reduce-scatter":
        outs = oracle.ring_reduce_scatter(case.inputs, case.eb, case.op, trace, raw=True)
    elif case.algo == "lossless-allgather":
        outs = oracle.ring_allgather(case.inputs, case.eb, trace, raw=True)
    else:
        outs = oracle.ring_allgather(case.inputs, case.eb, trace)
    assert len(outs) == case.N
    for o, e in zip(outs, case.outputs):
        assert np.asarray(o, np.float32).tobytes() == e.tobytes()
    assert [t[4] for t in trace] == case.msgs
    assert [t[2] for t in trace] == list(case.src) and [t[3] for t in trace] == list(case.dst)


SCAT = G.scatter_cases()


@pytest.mark.parametrize("case", SCAT, ids=[f"N{c.N}-root{c.root}" for c in SCAT])
def test_oracle_scatter_matches_reference(case, oracle):
    trace = []
    outs = oracle.binomial_scatter(case.data, case.N, 1e-4, root=case.root, counts=case.counts, trace=trace)
    for o, e in zip(outs, case.outputs):
        assert o.tobytes() == e.tobytes()
    assert [t[2] for t in trace] == case.msgs
    assert [t[0] for t in trace] == list(case.src) and [t[1] for t in trace] == list(case.dst)


FR = G.fixed_rate_cases()


@pytest.mark.parametrize("k", range(len(FR)))
def test_oracle_fixed_rate_matches_reference(k, oracle):
    x, b, blob, y = FR[k]
    assert oracle.fixed_rate_compress(x, b) == blob
    assert oracle.fixed_rate_decompress(blob).tobytes() == y.tobytes()


FRZ = G.fixed_rate_zero_cases()


@pytest.mark.parametrize("k", range(len(FRZ)))
def test_oracle_fixed_rate_signed_zero_extremum(k, oracle):
    # numpy's x.min()/x.max() pick a zero's sign by SIMD lane order (codec.py:454-455);
    # the oracle restates the AVX-512 reduction and must reproduce the reference's header
    x, b, blob, y = FRZ[k]
    assert oracle.fixed_rate_compress(x, b) == blob
    assert oracle.fixed_rate_decompress(blob).tobytes() == y.tobytes()


def test_avx512_extremum_model_matches_host_numpy(oracle):
    import math

    from numpy._core._multiarray_umath import __cpu_features__ as feats

    if not feats.get("AVX512_SKX"):
        pytest.skip("host numpy does not dispatch AVX-512: its signed-zero choice differs by design")
    rng = np.random.default_rng(11)
    for t in range(300):
        n = int(rng.integers(1, 700))
        x = (rng.integers(0, 2, n) * (1 if t % 2 else -1)).astype(np.float32)
        z = x == 0
        x[z] = np.where(rng.random(int(z.sum())) < 0.5, -0.0, 0.0)
        for op in ("min", "max"):
            ref = x.min() if op == "min" else x.max()
            got = oracle.np_extremum_avx512(x, op)
            assert got == ref and math.copysign(1, got) == math.copysign(1, ref), (n, op)
