"""The drop-in boundary for the collectives: the B200 transports plugged into
the REFERENCE's own algorithms and driver (gzccl from baseline/_ref, tests
only), and this package's run_collective against the reference's.

* every algorithm of the reference (collectives.py:540-553) run with
  GpuEbCodecTransport / GpuFixedRateTransport instead of the numpy transports
  gives byte-identical outputs, byte-identical traced messages, identical
  counters (with the default timing="model" even the simulated seconds) and
  identical transport totals;
* the reference's run_collective with ``make_transport`` replaced by ours
  returns the same report;
* our run_collective(network, ...) on the device fills the reference's
  Network counters / trace like simnet and reports the same counts,
  compression ratio and accuracy statistics.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "gzccl")):
    pytest.skip("reference package not installed in baseline/_ref", allow_module_level=True)
if REF not in sys.path:
    sys.path.append(REF)

from gzccl import collectives as RC  # noqa: E402
from gzccl import simnet as RS  # noqa: E402

from paper_2308_05199_b200 import collectives as C  # noqa: E402
from paper_2308_05199_b200 import transport as T  # noqa: E402


def _inputs(N, n, seed, scatter=False):
    rng = np.random.default_rng(seed)
    if scatter:
        return (np.sin(np.arange(n) / 37.0) + rng.normal(0, 0.01, n)).astype(np.float32)
    return [(np.sin(np.arange(n) / 37.0 + r) + rng.normal(0, 0.01, n)).astype(np.float32) for r in range(N)]


CASES = [
    ("ring-allreduce", 4, 5000, "sum"),
    ("ring-allreduce", 3, 777, "max"),
    ("ring-reduce-scatter", 5, 4099, "sum"),
    ("ring-allgather", 4, 1000, "sum"),
    ("rd-allreduce", 6, 3000, "sum"),
    ("rd-allreduce", 8, 2048, "max"),
    ("binomial-scatter", 7, 10000, None),
    ("cprp2p-allgather", 4, 999, None),
]


def _run_ref(algo, N, inputs, transport_factory, op, root=0):
    net = RS.Network(RS.CommunicatorSpec(N, root), record_payloads=True)
    tr = transport_factory(net.params)
    outs = RC.get_algorithm(algo).run(net, inputs, tr, reduce_op=op or "sum")
    return outs, net, tr


@pytest.mark.parametrize("codec", ["ebz", "fixed-rate"])
@pytest.mark.parametrize("algo,N,n,op", CASES, ids=[f"{a}-N{N}-n{n}-{op}" for a, N, n, op in CASES])
def test_device_transport_in_reference_algorithms(algo, N, n, op, codec):
    inputs = _inputs(N, n, N * n, scatter=algo == "binomial-scatter")
    eb, bits = 1e-4, 10
    ref_factory = (lambda p: RC.EbCodecTransport(p, eb)) if codec == "ebz" else (lambda p: RC.FixedRateTransport(p, bits))
    gpu_factory = (lambda p: T.GpuEbCodecTransport(p, eb)) if codec == "ebz" else (lambda p: T.GpuFixedRateTransport(p, bits))
    root = N // 2 if algo == "binomial-scatter" else 0
    ref_out, ref_net, ref_tr = _run_ref(algo, N, inputs, ref_factory, op, root)
    gpu_out, gpu_net, gpu_tr = _run_ref(algo, N, inputs, gpu_factory, op, root)
    for a, b in zip(ref_out, gpu_out):
        assert np.asarray(a, np.float32).tobytes() == np.asarray(b, np.float32).tobytes()
    assert [(s, d, ln, p) for s, d, ln, p in gpu_net.trace] == [(s, d, ln, p) for s, d, ln, p in ref_net.trace]
    for r0, r1 in zip(ref_net.ranks, gpu_net.ranks):
        assert r1.counters.as_dict() == r0.counters.as_dict()  # counts, bytes AND modelled seconds
        assert r1.clock == r0.clock
    assert (gpu_tr.raw_bytes_in, gpu_tr.blob_bytes_out) == (ref_tr.raw_bytes_in, ref_tr.blob_bytes_out)
    assert gpu_tr.name == ref_tr.name


@pytest.mark.parametrize("algo,codec", [("ring-allreduce", "ebz"), ("binomial-scatter", "ebz"),
                                        ("rd-allreduce", "fixed-rate"), ("lossless-allreduce", "ebz")])
def test_reference_run_collective_with_device_transports(algo, codec, monkeypatch):
    N, n = 4, 3000
    inputs = _inputs(N, n, 7, scatter=algo == "binomial-scatter")
    kw = dict(eb=1e-4, codec=codec, bits=9)
    ref_out, ref_rep = RS.run_collective(RS.Network(RS.CommunicatorSpec(N)), algo, inputs, **kw)
    monkeypatch.setattr(RC, "make_transport", T.make_transport)  # the one-line integration
    gpu_out, gpu_rep = RS.run_collective(RS.Network(RS.CommunicatorSpec(N)), algo, inputs, **kw)
    for a, b in zip(ref_out, gpu_out):
        assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    assert gpu_rep.to_dict() == ref_rep.to_dict()


REPORT_CASES = [("ring-allreduce", "ebz", 4), ("ring-reduce-scatter", "ebz", 3), ("ring-allgather", "ebz", 5),
                ("rd-allreduce", "ebz", 6), ("binomial-scatter", "ebz", 5), ("cprp2p-allgather", "ebz", 4),
                ("ring-allreduce", "fixed-rate", 4), ("rd-allreduce", "fixed-rate", 3),
                ("binomial-scatter", "fixed-rate", 4), ("lossless-allreduce", "ebz", 4),
                ("lossless-scatter", "ebz", 3), ("ring-allreduce", "none", 4)]


@pytest.mark.parametrize("algo,codec,N", REPORT_CASES, ids=[f"{a}-{c}-N{N}" for a, c, N in REPORT_CASES])
def test_run_collective_matches_reference_report(algo, codec, N):
    n = 2500
    sc = C.get_algorithm(algo).family == "scatter"
    inputs = _inputs(N, n, 11 * N, scatter=sc)
    kw = dict(eb=1e-4, codec=codec, bits=11, reduce_op="sum")
    ref_net = RS.Network(RS.CommunicatorSpec(N, N - 1 if sc else 0), record_payloads=True)
    ref_out, ref_rep = RS.run_collective(ref_net, algo, inputs, **kw)
    net = RS.Network(RS.CommunicatorSpec(N, N - 1 if sc else 0), record_payloads=True)
    out, rep = C.run_collective(net, algo, inputs, **kw)  # device execution, reference network object
    for a, b in zip(ref_out, out):
        assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    assert [(s, d, ln, p) for s, d, ln, p in net.trace] == [(s, d, ln, p) for s, d, ln, p in ref_net.trace]
    for key in ("n_compress", "n_decompress", "n_messages", "bytes_sent", "bytes_received"):
        assert rep.counters[key] == ref_rep.counters[key], key
        assert [c[key] for c in rep.counters_per_rank] == [c[key] for c in ref_rep.counters_per_rank], key
    for r0, r1 in zip(ref_net.ranks, net.ranks):
        assert r1.counters.n_compress == r0.counters.n_compress
    assert rep.compression_ratio == ref_rep.compression_ratio
    assert (rep.algorithm, rep.ranks, rep.root, rep.elements_per_rank, rep.total_elements, rep.eb, rep.codec,
            rep.reduce_op) == (ref_rep.algorithm, ref_rep.ranks, ref_rep.root, ref_rep.elements_per_rank,
                               ref_rep.total_elements, ref_rep.eb, ref_rep.codec, ref_rep.reduce_op)
    a, b = rep.accuracy, ref_rep.accuracy
    assert a.max_abs_err == b.max_abs_err
    assert a.mse == pytest.approx(b.mse, rel=1e-12, abs=0)
    assert a.mean_signed_err == pytest.approx(b.mean_signed_err, rel=1e-9, abs=1e-18)
    assert (a.psnr == b.psnr) if np.isinf(b.psnr) else a.psnr == pytest.approx(b.psnr, rel=1e-12)
    d = rep.to_dict()
    assert d["schema"] == "gzccl.report.v1" and set(ref_rep.to_dict()) <= set(d)


def test_run_collective_nonfinite_and_errors():
    bad = [np.ones(100, np.float32) for _ in range(3)]
    bad[1][42] = np.nan
    bad[2][7] = np.inf
    with pytest.raises(ValueError, match="non-finite value at offset 42"):
        C.run_collective(3, "ring-allreduce", bad, eb=1e-4)
    with pytest.raises(ValueError, match="error bound"):
        C.run_collective(3, "ring-allreduce", [np.ones(4, np.float32)] * 3)
    with pytest.raises(ValueError, match="unknown codec"):
        C.run_collective(3, "ring-allreduce", [np.ones(4, np.float32)] * 3, eb=1e-4, codec="zfp")
    with pytest.raises(ValueError, match="error bound"):
        T.make_transport("ebz", RS.Network(RS.CommunicatorSpec(2)).params)
