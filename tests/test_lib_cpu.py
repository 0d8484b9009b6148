"""CPU-only checks: the C-ABI library loads and exports every symbol
include/gzccl.h declares; host-side helpers (no device compute)."""

import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "gzccl.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|uint32_t|void)\s+(gz_[a-z0-9_]+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "gz_compress" in syms and "gz_reduce_step" in syms and len(syms) >= 20


def test_library_loads_and_exports_everything():
    from paper_2308_05199_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2308_05199_b200 import build

        build.build()
    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_host_sizing_functions():
    from paper_2308_05199_b200 import _lib

    L = _lib.lib()
    tb = L.gz_tile_blocks()
    assert tb in (32, 64, 128, 256)
    for n in (0, 1, 31, 32, 33, 4096, 1 << 24, (1 << 24) + 5):
        nb = -(-n // 32)
        assert L.gz_compress_bound(n) >= 24 + nb * 129
        assert L.gz_num_tiles(n) == -(-nb // tb)
        assert L.gz_sidecar_bytes(n) % 16 == 0
    # argument checking paths that never touch the device
    assert L.gz_compress(None, 10, 1e-4, 64, None, 0, None, None, None, None, 0, None, None) == _lib.GZ_EBLOCK
    assert L.gz_compress(None, 10, -1.0, 32, None, 0, None, None, None, None, 0, None, None) == _lib.GZ_EBOUND
    assert L.gz_compress(None, 10, 1e-4, 32, None, 0, None, None, None, None, 0, None, None) == _lib.GZ_EINVAL
    # flag batches: empty, oversized and null-pointer batches are refused before any driver call
    from paper_2308_05199_b200.comm import _FlagOp

    ops = (_FlagOp * 65)()
    assert L.gz_stream_flag_ops(None, ops, 0) == _lib.GZ_EINVAL
    assert L.gz_stream_flag_ops(None, ops, 65) == _lib.GZ_EINVAL
    assert L.gz_stream_flag_ops(None, ops, 1) == _lib.GZ_EINVAL  # ptr NULL
    bad = (_FlagOp * 1)(_FlagOp(0x1000, 1, 7))  # unknown kind
    assert L.gz_stream_flag_ops(None, bad, 1) == _lib.GZ_EINVAL


def test_chunk_spans_and_tree_match_reference_semantics(oracle):
    from paper_2308_05199_b200 import collectives as C

    for n in (0, 1, 5, 16, 17, 100):
        for N in (1, 2, 3, 7, 16):
            assert C.chunk_spans(n, N) == oracle.chunk_spans(n, N)
    for N in range(1, 40):
        for vr in range(N):
            assert C.scatter_children(vr, N) == oracle.scatter_children(vr, N)
    assert C.scatter_msg_overhead(8) == 24 + 64


def test_package_refuses_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_2308_05199_b200 as gz

    with pytest.raises(RuntimeError, match="CUDA"):
        gz.compress(np.zeros(10, np.float32), 1e-4)
