"""Packing paths of the encoder (csrc/gz_codec.cu encode_tile): warp tiles whose 32
blocks are all full, packed and of width <= 4 take the one-shot `pack_small`
assembly, every other tile the streaming Appender.  Inputs are engineered block by
block (target code width 0..8, raw blocks, partial tiles) so that both paths, and
tiles that mix them at the boundary, are compared byte for byte with the CPU
oracle (codec.py:244-270) -- for the plain compressor and for the fused reduce-
scatter step of a virtual ring allreduce (collectives.py:258-308)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_05199_b200 as gz  # noqa: E402
from paper_2308_05199_b200 import collectives as C  # noqa: E402

TILE_BLOCKS = 32


def engineered(widths, eb, rng, raw_blocks=(), tail=0):
    """One 32-value block per entry of `widths`: a random start and 31 steps of
    k * 2 eb with the zigzag code of k below 2^w (w = 0: a constant block)."""
    tw = 2.0 * eb
    out = []
    for b, w in enumerate(widths):
        x0 = rng.uniform(-1.0, 1.0)
        if w == 0:
            k = np.zeros(31)
        else:
            k = rng.integers(-(1 << (w - 1)), 1 << (w - 1), 31).astype(np.float64)
        blk = x0 + tw * np.concatenate([[0.0], np.cumsum(k)])
        if b in raw_blocks:
            blk[17] += 1e12  # |q| > 2^30: codec.py:201-202 stores the block raw
        out.append(blk)
    x = np.concatenate(out).astype(np.float32)
    if tail:
        x = np.concatenate([x, rng.uniform(-1, 1, tail).astype(np.float32)])
    return x


def patterns(rng):
    tiles = 24
    nb = tiles * TILE_BLOCKS
    yield "all_w_le_4", rng.integers(0, 5, nb), (), 0
    yield "all_w4", np.full(nb, 4), (), 0
    yield "all_w0", np.zeros(nb, int), (), 0
    mixed = rng.integers(0, 5, nb)
    mixed[5 * TILE_BLOCKS + 31] = 5  # the last block of tile 5 pushes it to the Appender
    mixed[9 * TILE_BLOCKS] = 8       # the first block of tile 9
    mixed[11 * TILE_BLOCKS + 16] = 6
    yield "boundary_w5_w8", mixed, (), 0
    yield "raw_blocks", rng.integers(0, 5, nb), (3 * TILE_BLOCKS + 7, 20 * TILE_BLOCKS + 31), 0
    yield "wide", rng.integers(0, 9, nb), (), 0
    yield "partial_tail", rng.integers(0, 5, nb), (), 517


@pytest.fixture(scope="module")
def ws():
    return gz.Workspace()


@pytest.mark.parametrize("eb", [1e-4, 3.7e-3])
def test_pack_paths_compress(eb, oracle, ws):
    rng = np.random.default_rng(11)
    for name, widths, raw, tail in patterns(rng):
        x = engineered(widths, eb, rng, raw, tail)
        ref = oracle.compress(x, eb, threads=8)
        blob = gz.compress(torch.from_numpy(x).cuda(), eb, ws)
        assert bytes(blob) == ref, name
        assert gz.decompress(blob, ws).cpu().numpy().tobytes() == oracle.decompress(ref, threads=8).tobytes(), name


@pytest.mark.parametrize("N", [2, 3])
def test_pack_paths_fused_step(N, oracle, ws):
    # the fused reduce-scatter step encodes op(local, decoded) with the same packing
    rng = np.random.default_rng(5 + N)
    eb = 1e-4
    for name, widths, raw, tail in patterns(rng):
        bufs = [engineered(widths, eb, rng, raw, tail) for _ in range(N)]
        ref = oracle.ring_allreduce([b.copy() for b in bufs], eb, threads=8)
        got = C.ring_allreduce_virtual([torch.from_numpy(b).cuda() for b in bufs], eb, ws=ws)
        for r in range(N):
            assert got[r].cpu().numpy().tobytes() == np.asarray(ref[r], np.float32).tobytes(), (name, r)
