"""Cost model (costmodel.py): the restated timelines equal the reference's
predicted_makespan for every algorithm, rank count and behaviour flag, the
parameter semantics follow costmodel.py:31-134, and the B200 fit (when
profiles/b200_cost_params.json exists) loads and predicts the measured ring
allreduce within its recorded tolerance.  CPU only."""

import itertools
import json
import math
import os
import sys

import pytest

from paper_2308_05199_b200 import costmodel as M

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.path.join(ROOT, "baseline", "_ref")

ALGOS = ["ring-allgather", "ring-reduce-scatter", "ring-allreduce", "rd-allreduce", "binomial-scatter",
         "cprp2p-allgather", "lossless-allgather", "lossless-reduce-scatter", "lossless-allreduce", "lossless-scatter"]


def _ref():
    if not os.path.isdir(os.path.join(REF, "gzccl")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.append(REF)
    from gzccl import costmodel as RM

    return RM


@pytest.mark.parametrize("overlap,staging,multi", list(itertools.product([False, True], repeat=3)))
def test_predicted_makespan_matches_reference(overlap, staging, multi):
    RM = _ref()
    kw = dict(alpha=3e-6, beta=1.3e-12, launch=7e-6, saturation=2.5e6, compress_throughput=2.6e12,
              decompress_throughput=4.1e12, reduce_throughput=5e12, host_device_bandwidth=5.5e10,
              staging=staging, overlap=overlap, multi_stream=multi)
    ours, theirs = M.CostParams(**kw), RM.CostParams(**kw)
    for algo in ALGOS:
        for N in (1, 2, 3, 4, 5, 6, 7, 8, 12, 16):
            for D in (1e3, 3e6, 5.4e8):
                for cr in (1.0, 7.1, 64.0):
                    a = M.predicted_makespan(algo, D, N, ours, cr)
                    b = RM.predicted_makespan(algo, D, N, theirs, cr)
                    assert a == pytest.approx(b, rel=1e-12, abs=1e-18), (algo, N, D, cr)


def test_default_params_and_crossover_match_reference():
    RM = _ref()
    for algo in ALGOS:
        for N in (2, 8, 64):
            assert M.predicted_makespan(algo, 1e8, N) == pytest.approx(RM.predicted_makespan(algo, 1e8, N), rel=1e-12)
    # test_costmodel.py:155-176: at 646 MB ring wins at 8 ranks, recursive doubling from 64..256 ranks on
    D = 646e6
    assert M.predicted_makespan("ring-allreduce", D, 8) < M.predicted_makespan("rd-allreduce", D, 8)
    ns = range(2, 2049)
    ring = {n: M.predicted_makespan("ring-allreduce", D, n) for n in ns}
    rd = {n: M.predicted_makespan("rd-allreduce", D, n) for n in ns}
    n_star = next(n for n in ns if all(rd[m] < ring[m] for m in ns if m >= n))
    assert 64 <= n_star <= 256


def test_parameter_semantics():
    p = M.CostParams()
    assert p.msg_time(0) == p.alpha
    assert p.kernel_time(0, "compress") == p.kernel_time(p.saturation, "compress")  # plateau
    assert p.kernel_time(2 * p.saturation, "compress") > p.kernel_time(p.saturation, "compress")
    assert p.staging_time(1e9) == 0.0
    assert M.CostParams(staging=True).staging_time(1.0) == pytest.approx(2.0 / p.host_device_bandwidth)
    assert M.CostParams(overlap=True).step_time(3.0, 4.0) == 4.0 and p.step_time(3.0, 4.0) == 7.0
    q = M.CostParams(multi_stream=True)
    assert q.multi_launch_time([1e6] * 64, "compress") <= p.multi_launch_time([1e6] * 64, "compress")
    for bad in (dict(alpha=0), dict(beta=-1.0), dict(launch=float("inf")), dict(saturation=float("nan"))):
        with pytest.raises(ValueError):
            M.CostParams(**bad)
    with pytest.raises(ValueError, match="unknown kernel kind"):
        p.kernel_time(1, "decode")
    with pytest.raises(ValueError):
        p.msg_time(-1)
    with pytest.raises(ValueError):
        p.multi_launch_time([], "compress")
    with pytest.raises(ValueError):
        M.predicted_makespan("ring-allreduce", 0, 8)
    with pytest.raises(ValueError):
        M.predicted_makespan("ring-allreduce", 1e6, 0)
    with pytest.raises(ValueError, match="unknown algorithm"):
        M.predicted_makespan("warp-drive", 1e6, 8)


def test_load_round_trip(tmp_path):
    p = M.CostParams(alpha=2e-6, overlap=True)
    f = tmp_path / "c.json"
    f.write_text(json.dumps(p.to_dict()))
    assert M.load_cost_params(str(f)) == p
    assert M.load_cost_params(None, beta=1e-12).beta == 1e-12
    f.write_text(json.dumps({"gamma": 1}))
    with pytest.raises(ValueError, match="unknown cost parameter"):
        M.load_cost_params(str(f))


FIT = os.path.join(ROOT, "profiles", "b200_cost_params.json")


@pytest.mark.skipif(not os.path.exists(FIT), reason="no B200 fit committed yet")
def test_b200_fit_predicts_measured_allreduce():
    d = json.load(open(FIT))
    p = M.b200_cost_params(FIT)
    assert p.overlap and not p.staging
    for row in d["checks"]:
        pred = M.predicted_makespan(row["algorithm"], row["bytes"], row["ranks"], p, row["cr"])
        assert math.isfinite(pred) and pred > 0
        assert pred == pytest.approx(row["predicted_s"], rel=1e-9)
        assert abs(pred / row["measured_s"] - 1.0) <= d["tolerance"], row
