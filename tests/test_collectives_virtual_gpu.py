"""Collective schedules with N virtual ranks on one GPU vs the reference's own
outputs and traced messages (golden fixtures) -- bit-exact."""

import numpy as np
import pytest

import golden_data as G
from conftest import max_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_05199_b200 as gz  # noqa: E402
from paper_2308_05199_b200 import collectives as C  # noqa: E402

RING = G.ring_cases()


@pytest.fixture(scope="module")
def ws():
    return gz.Workspace()


def _np(o):
    return o.cpu().numpy() if isinstance(o, torch.Tensor) else np.asarray(o)


@pytest.mark.parametrize("case", RING, ids=[f"{c.algo}-N{c.N}-n{c.n}-{c.op}" for c in RING])
def test_ring_matches_reference(case, ws):
    net = C.create_network(C.CommunicatorSpec(case.N), record_payloads=True)
    outs, rep = C.run_collective(net, case.algo, case.inputs, eb=case.eb, reduce_op=case.op, workspace=ws)
    assert len(outs) == case.N
    for o, e in zip(outs, case.outputs):
        assert _np(o).tobytes() == e.tobytes()
    msgs = net.trace
    assert [m[3] for m in msgs] == case.msgs
    assert [m[2] for m in msgs] == [len(b) for b in case.msgs]
    assert [m[0] for m in msgs] == list(case.src) and [m[1] for m in msgs] == list(case.dst)


SCAT = G.scatter_cases()


@pytest.mark.parametrize("case", SCAT, ids=[f"N{c.N}-root{c.root}" for c in SCAT])
def test_scatter_matches_reference(case, ws):
    net = C.create_network(C.CommunicatorSpec(case.N, case.root), record_payloads=True)
    outs, rep = C.run_collective(net, "binomial-scatter", case.data, eb=1e-4, counts=case.counts, workspace=ws)
    for o, e in zip(outs, case.outputs):
        assert _np(o).tobytes() == e.tobytes()
    assert [m[3] for m in net.trace] == case.msgs
    assert [m[0] for m in net.trace] == list(case.src)
    assert [m[1] for m in net.trace] == list(case.dst)


OP_COUNT_CASES = [
    ("ring-reduce-scatter", lambda N: (N - 1, N - 1)),
    ("ring-allgather", lambda N: (1, N - 1)),
    ("ring-allreduce", lambda N: (N, 2 * (N - 1))),
]


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("algo,expect", OP_COUNT_CASES)
def test_op_counts(algo, expect, N, ws):
    # pkg/tests/test_collectives.py:61-80
    rng = np.random.default_rng(N)
    inputs = [rng.uniform(0, 1, 2 * N).astype(np.float32) for _ in range(N)]
    _, rep = C.run_collective(N, algo, inputs, eb=1e-4, workspace=ws)
    for c in rep.counters_per_rank:
        assert (c["n_compress"], c["n_decompress"]) == expect(N)


@pytest.mark.parametrize("eb", [1e-3, 1e-4, 1e-5])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_allreduce_error_budget(eb, N, oracle, ws):
    # README error budgets: ring allreduce <= N * eb vs the lossless ring
    rng = np.random.default_rng(int(N / eb) % 1000)
    n = 50_000
    inputs = [oracle.smooth_field(n, 0.37 * r) + rng.normal(0, 1e-2, n).astype(np.float32) for r in range(N)]
    outs, _ = C.run_collective(N, "ring-allreduce", inputs, eb=eb, workspace=ws)
    lossless = oracle.ring_allreduce(inputs, eb, raw=True)
    for o, e in zip(outs, lossless):
        assert max_err(e, _np(o)) <= N * eb


def test_errors(ws):
    with pytest.raises(ValueError, match="equal length"):
        C.run_collective(2, "ring-allreduce", [np.zeros(10, np.float32), np.zeros(11, np.float32)], eb=1e-4, workspace=ws)
    with pytest.raises(ValueError, match="counts"):
        C.run_collective(2, "binomial-scatter", np.zeros(10, np.float32), eb=1e-4, counts=[4, 4], workspace=ws)
    with pytest.raises(ValueError, match="unknown algorithm"):
        C.run_collective(1, "nope", [np.zeros(4, np.float32)], eb=1e-4)
    with pytest.raises(ValueError, match="unknown reduce op"):
        C.run_collective(2, "ring-allreduce", [np.zeros(4, np.float32)] * 2, eb=1e-4, reduce_op="prod", workspace=ws)


def test_zero_preservation(ws):
    zeros = [np.zeros(64, np.float32) for _ in range(4)]
    for algo in ("ring-allgather", "ring-reduce-scatter", "ring-allreduce"):
        outs, _ = C.run_collective(4, algo, zeros, eb=1e-4, workspace=ws)
        for o in outs:
            assert np.all(_np(o) == 0.0)


@pytest.mark.parametrize("N", [2, 4, 8, 16])
def test_rd_power_of_two_op_counts(N, ws):
    # pkg/tests/test_collectives.py:78-84
    k = N.bit_length() - 1
    rng = np.random.default_rng(N)
    inputs = [rng.uniform(0, 1, 64).astype(np.float32) for _ in range(N)]
    _, rep = C.run_collective(N, "rd-allreduce", inputs, eb=1e-4, workspace=ws)
    for c in rep.counters_per_rank:
        assert (c["n_compress"], c["n_decompress"]) == (k, k)


@pytest.mark.parametrize("N", [3, 6, 12])
def test_rd_remainder_roles(N, ws):
    # pkg/tests/test_collectives.py:86-99
    pof2, r, k, role, _, _ = C.rd_plan(N)
    rng = np.random.default_rng(N)
    inputs = [rng.uniform(0, 1, 64).astype(np.float32) for _ in range(N)]
    _, rep = C.run_collective(N, "rd-allreduce", inputs, eb=1e-4, workspace=ws)
    for i, c in enumerate(rep.counters_per_rank):
        got = (c["n_compress"], c["n_decompress"])
        assert got == {"donor": (1, 1), "absorber": (k + 1, k + 1), "direct": (k, k)}[role(i)]


@pytest.mark.parametrize("eb", [1e-2, 1e-3, 1e-4])
@pytest.mark.parametrize("N", [3, 4, 6, 7, 8])
def test_rd_error_budget(eb, N, oracle, ws):
    # pkg/tests/test_collectives.py:140-154: (N-1) eb at powers of two, 2 N eb otherwise
    bound = (N - 1) * eb if N & (N - 1) == 0 else 2 * N * eb
    for seed in range(3):
        rng = np.random.default_rng(50 * seed + N)
        bufs = [rng.uniform(0, 1, 60).astype(np.float32) for _ in range(N)]
        outs, _ = C.run_collective(N, "rd-allreduce", bufs, eb=eb, workspace=ws)
        lossless = oracle.rd_allreduce(bufs, eb, raw=True)
        for o, e in zip(outs, lossless):
            assert max_err(e, _np(o)) <= bound


def _synth_images(images, width, height, seed):
    # gzccl cli.py:170-181 (cfg5 image stacking input)
    yy, xx = np.mgrid[0:height, 0:width]
    base = 0.5 + 0.25 * np.sin(2 * np.pi * 3 * xx / width) * np.cos(2 * np.pi * 2 * yy / height)
    rng = np.random.default_rng(seed)
    return [np.clip(base + rng.uniform(-0.2, 0.2, base.shape), 0.0, 1.0).astype(np.float32).ravel()
            for _ in range(images)]


@pytest.mark.parametrize("eb,cr,psnr_db,maxerr", [(2e-4, 2.39, 85.7, 1.34e-3), (1e-4, 2.22, 91.7, 6.48e-4)])
def test_image_stacking_cfg5(eb, cr, psnr_db, maxerr, oracle, ws):
    # BASELINE.md section 2 (reference measured here): 8 images 512x512, ring-allreduce sum;
    # outputs bit-exact with the oracle, so CR / PSNR / max error reproduce the reference's
    imgs = _synth_images(8, 512, 512, 0)
    outs, rep = C.run_collective(8, "ring-allreduce", imgs, eb=eb, workspace=ws)
    expect = oracle.ring_allreduce(imgs, eb)
    for o, e in zip(outs, expect):
        assert _np(o).tobytes() == e.tobytes()
    ref = np.concatenate(oracle.ring_allreduce(imgs, eb, raw=True)).astype(np.float64)
    got = np.concatenate([_np(o) for o in outs]).astype(np.float64)
    err = np.abs(ref - got)
    mse = float(np.mean((ref - got) ** 2))
    rng_ = float(ref.max() - ref.min())
    assert rep.compression_ratio == pytest.approx(cr, abs=0.01)
    assert 10 * np.log10(rng_ ** 2 / mse) == pytest.approx(psnr_db, abs=0.05)
    assert float(err.max()) == pytest.approx(maxerr, rel=0.01)
    assert float(err.max()) <= 8 * eb
    # the report's own accuracy block: the lossless rerun of the same schedule on the device
    assert rep.accuracy.max_abs_err == pytest.approx(float(err.max()), rel=1e-12)
    assert rep.accuracy.psnr == pytest.approx(psnr_db, abs=0.05)


def test_lossless_scatter_exact(ws):
    rng = np.random.default_rng(5)
    data = rng.normal(0, 1, 1000).astype(np.float32)
    outs, _ = C.run_collective(4, "lossless-scatter", data, counts=[100, 200, 300, 400], workspace=ws)
    lo = 0
    for o, c in zip(outs, [100, 200, 300, 400]):
        assert _np(o).tobytes() == data[lo:lo + c].tobytes()
        lo += c


@pytest.mark.parametrize("N", [2, 4, 7])
def test_cprp2p_hop_error(N, oracle, ws):
    # collectives.py:311-316: a chunk that travelled h hops carries up to h * eb
    eb = 1e-3
    rng = np.random.default_rng(N)
    chunks = [rng.uniform(0, 1, 100).astype(np.float32) for _ in range(N)]
    outs, rep = C.run_collective(N, "cprp2p-allgather", chunks, eb=eb, workspace=ws)
    for i, o in enumerate(outs):
        o = _np(o)
        for c in range(N):
            h = (i - c) % N
            assert np.max(np.abs(o[100 * c:100 * (c + 1)] - chunks[c])) <= max(h, 0) * eb + 1e-7
    for cnt in rep.counters_per_rank:
        assert (cnt["n_compress"], cnt["n_decompress"]) == (N - 1, N - 1)
