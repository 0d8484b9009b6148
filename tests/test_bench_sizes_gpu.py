"""Parity at the benchmark sizes (BASELINE.json configs), bit-exact vs the CPU oracle.

The bench lines time the codec on 2^24 and 2^27 values, the ring allreduce on
512 MiB (2^27 f32) per rank and the binomial scatter on a 1 GiB (2^28 f32)
root buffer.  These tests run the same kernels at those sizes -- the fused
reduce-scatter step, the multi-owner allgather decode and the multi-segment
scatter root included -- with all N ranks on one GPU (the reference's own
two-pass schedule, collectives.py:258-308, 467-532) and compare every byte of
every rank's output with the oracle run on all host threads.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_05199_b200 as gz  # noqa: E402
from paper_2308_05199_b200 import collectives as C  # noqa: E402

EB = 1e-4
CFG2 = 1 << 27  # 512 MiB of f32 per rank
CFG3 = 1 << 28  # 1 GiB of f32 at the scatter root


def threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


@pytest.fixture(scope="module")
def ws():
    return gz.Workspace()


@pytest.mark.parametrize("n", [1 << 24, 1 << 27])
def test_codec_at_bench_sizes(n, oracle, ws):
    # bench.py N=1: cfg1 (2^24) and the 2^27 supplementary field
    x = oracle.smooth_field(n)
    ref, offs = oracle.compress(x, EB, threads=threads(), return_offsets=True)
    blob = gz.compress(torch.from_numpy(x).cuda(), EB, ws, return_offsets=True)
    assert len(blob) == len(ref)
    assert blob.data.cpu().numpy().tobytes() == ref
    assert np.array_equal(blob.block_offsets.cpu().numpy(), offs.astype(np.int64))
    y = gz.decompress(blob, ws)
    assert y.cpu().numpy().tobytes() == oracle.decompress(ref, threads=threads()).tobytes()


@pytest.mark.parametrize("N,per_rank", [(2, CFG2), (4, CFG2), (8, 1 << 25)])
def test_ring_allreduce_at_cfg2_scale(N, per_rank, oracle, ws):
    # configs[1]: ring allreduce, smooth field per rank with phase 0.37 r (bench.py N>1)
    bufs = [oracle.smooth_field(per_rank, 0.37 * r) for r in range(N)]
    expect = oracle.ring_allreduce(bufs, EB, threads=threads())
    outs = C.ring_allreduce_virtual(bufs, EB, ws=ws)
    for r in range(N):
        got = outs[r].cpu().numpy()
        assert got.tobytes() == expect[r].tobytes(), f"rank {r} differs"
    del outs, expect


@pytest.mark.parametrize("N", [2, 8])
def test_binomial_scatter_at_cfg3_scale(N, oracle, ws):
    # configs[2]: 1 GiB root buffer (2^28 f32), chunk_spans counts, root 0
    data = oracle.smooth_field(CFG3, 0.0)
    expect = oracle.binomial_scatter(data, N, EB, root=0, threads=threads())
    outs = C.binomial_scatter_virtual(data, N, EB, root=0, ws=ws)
    for r in range(N):
        assert outs[r].cpu().numpy().tobytes() == expect[r].tobytes(), f"rank {r} differs"
