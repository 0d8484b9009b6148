"""Device codec parity: libgzccl.so kernels vs the reference (golden fixtures)
and vs the CPU oracle on seeded inputs.  Bit-exact bytes, offsets, outputs."""

import hashlib

import numpy as np
import pytest

import golden_data as G
from conftest import max_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2308_05199_b200 as gz  # noqa: E402

CASES = G.codec_cases()


@pytest.fixture(scope="module")
def ws():
    return gz.Workspace()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_compress_bytes_and_offsets_match_reference(case, ws):
    x = torch.from_numpy(case.x).cuda()
    blob = gz.compress(x, case.eb, ws, return_offsets=True)
    assert bytes(blob) == case.blob
    if case.x.size:
        assert np.array_equal(blob.block_offsets.cpu().numpy(), case.block_offsets)


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_decompress_sidecar_matches_reference(case, ws):
    blob = gz.compress(torch.from_numpy(case.x).cuda(), case.eb, ws)
    y = gz.decompress(blob, ws)
    assert y.cpu().numpy().tobytes() == case.y.tobytes()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_decompress_reference_blob(case, ws):
    # a blob produced by the reference, decoded on the device (gz_index path)
    y = gz.decompress(case.blob, ws)
    assert isinstance(y, np.ndarray)
    assert y.tobytes() == case.y.tobytes()


def test_host_api_returns_bytes(ws):
    data, eb = G.golden_data(2)
    out = gz.compress(data, eb)
    assert isinstance(out, bytes) and out == G.golden_blob(2)
    back = gz.decompress(out)
    assert isinstance(back, np.ndarray) and max_err(data, back) <= eb


@pytest.mark.parametrize("seed", range(6))
def test_random_vs_oracle(seed, oracle, ws):
    rng = np.random.default_rng(seed)
    for _ in range(6):
        n = int(rng.integers(1, 300_000))
        kind = rng.integers(0, 4)
        if kind == 0:
            x = rng.uniform(-1, 1, n).astype(np.float32)
        elif kind == 1:
            x = np.cumsum(rng.normal(0, 1e-3, n)).astype(np.float32)
        elif kind == 2:
            x = (rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-6, 6, n)).astype(np.float32)
        else:
            x = oracle.smooth_field(n, float(seed))
        eb = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 3.7e-4]))
        ref = oracle.compress(x, eb, threads=8)
        blob = gz.compress(torch.from_numpy(x).cuda(), eb, ws)
        assert bytes(blob) == ref
        assert gz.decompress(blob, ws).cpu().numpy().tobytes() == oracle.decompress(ref, threads=8).tobytes()


@pytest.mark.parametrize("eb", [1e-4, 1e-3, 1e-2])
def test_cfg1_field_bit_exact(eb, oracle, ws):
    n = 1 << 24
    x = oracle.smooth_field(n)
    ref, offs = oracle.compress(x, eb, threads=8, return_offsets=True)
    blob = gz.compress(torch.from_numpy(x).cuda(), eb, ws, return_offsets=True)
    assert len(blob) == len(ref)
    assert bytes(blob) == ref
    assert np.array_equal(blob.block_offsets.cpu().numpy(), offs)
    d = G.digests()
    if hashlib.sha256(x.tobytes()).hexdigest() == d["cfg1_input_sha256"]:
        assert hashlib.sha256(ref).hexdigest() == d[f"cfg1_eb{eb!r}"]["sha256"]
    y = gz.decompress(blob, ws).cpu().numpy()
    assert y.tobytes() == oracle.decompress(ref, threads=8).tobytes()
    assert max_err(x, y) <= eb


def test_unaligned_and_offset_views(oracle, ws):
    base = torch.from_numpy(oracle.smooth_field(100_003)).cuda()
    for off in (1, 2, 3, 5, 31, 33):
        v = base[off:]
        assert bytes(gz.compress(v, 1e-4, ws)) == oracle.compress(base[off:].cpu().numpy(), 1e-4)


def test_errors(ws):
    with pytest.raises(ValueError, match="offset 2"):
        gz.compress(torch.tensor([0.0, 1.0, float("nan")], device="cuda"), 1e-4, ws)
    with pytest.raises(ValueError, match="offset 0"):
        gz.compress(np.array([np.inf], np.float32), 1e-4)
    x = np.zeros(100, np.float32)
    x[77] = -np.inf
    with pytest.raises(ValueError, match="offset 77"):
        gz.compress(x, 1e-4)
    for eb in (0.0, -1e-4, float("nan"), float("inf")):
        with pytest.raises(ValueError):
            gz.compress(np.ones(4, np.float32), eb)
    with pytest.raises(ValueError):
        gz.compress(np.ones(64, np.float32), 1e-4, block=64)
    blob = gz.compress(np.zeros(64, np.float32), 1e-4)
    with pytest.raises(gz.DecodeError, match="trailing"):
        gz.decompress(blob + b"\x00")
    bad = bytearray(blob)
    bad[24] = 77
    with pytest.raises(gz.DecodeError, match="width"):
        gz.decompress(bytes(bad))
    with pytest.raises(gz.DecodeError, match="magic"):
        gz.decompress(b"XXXX" + blob[4:])
    with pytest.raises(gz.DecodeError):
        gz.decompress(b"GZC1\x00\x00")
    b2 = gz.compress(np.random.default_rng(0).uniform(0, 1, 100).astype(np.float32), 1e-4)
    with pytest.raises(gz.DecodeError, match="truncated"):
        gz.decompress(b2[:-3])


def test_compress_blocks_and_decompress_block(ws):
    rng = np.random.default_rng(3)
    counts = [100, 2000, 4, 1992, 0]
    data = rng.uniform(0, 1, sum(counts)).astype(np.float32)
    payload, table = gz.compress_blocks(data, counts, 1e-4)
    import oracle.oracle as O

    expect = b"".join(O.compress(data[sum(counts[:i]) : sum(counts[: i + 1])], 1e-4) for i in range(len(counts)))
    assert payload == expect
    assert table.sizes[4] == 24
    pos = 0
    for i, c in enumerate(counts):
        got = gz.decompress_block(payload, table, i)
        assert got.size == c
        assert max_err(data[pos : pos + c], got) <= 1e-4
        pos += c
    with pytest.raises(IndexError):
        gz.decompress_block(payload, table, 5)
    with pytest.raises(ValueError, match="sum"):
        gz.compress_blocks(np.zeros(10, np.float32), [4, 4], 1e-4)
    with pytest.raises(ValueError, match="chain"):
        gz.BlockTable(sizes=(3, 4), offsets=(0, 5))


def test_many_segments_one_launch(oracle, ws):
    rng = np.random.default_rng(11)
    counts = [int(c) for c in rng.integers(0, 20000, 70)]
    data = oracle.smooth_field(sum(counts), 0.3)
    payload, table = gz.compress_blocks(data, counts, 1e-3)
    pos = 0
    for i, c in enumerate(counts):
        assert payload[table.offsets[i] : table.offsets[i] + table.sizes[i]] == oracle.compress(data[pos : pos + c], 1e-3)
        pos += c


def test_workspace_reuse_and_determinism(ws, oracle):
    x = torch.from_numpy(oracle.smooth_field(777_777)).cuda()
    a = bytes(gz.compress(x, 1e-4, ws))
    for _ in range(5):
        assert bytes(gz.compress(x, 1e-4, ws)) == a
    assert bytes(gz.compress(x, 1e-4, gz.Workspace())) == a


FR = G.fixed_rate_cases()


@pytest.mark.parametrize("k", range(len(FR)))
def test_fixed_rate_matches_reference(k, ws):
    # codec.py:442-489 (the comparator), byte-identical blobs and values
    x, b, blob, y = FR[k]
    assert gz.fixed_rate_compress(x, b, ws) == blob
    assert gz.fixed_rate_decompress(blob, ws).tobytes() == y.tobytes()
    dev = gz.fixed_rate_compress(torch.from_numpy(x).cuda(), b, ws)
    assert dev.cpu().numpy().tobytes() == blob
    assert gz.fixed_rate_decompress(dev, ws).cpu().numpy().tobytes() == y.tobytes()


FRZ = G.fixed_rate_zero_cases()


@pytest.mark.parametrize("k", range(len(FRZ)))
def test_fixed_rate_signed_zero_extremum(k, ws):
    # a zero min / max carries the sign numpy's AVX-512 reduction returns (codec.py:454-455)
    x, b, blob, y = FRZ[k]
    assert gz.fixed_rate_compress(x, b, ws) == blob
    assert gz.fixed_rate_decompress(blob, ws).tobytes() == y.tobytes()


def test_fixed_rate_errors(ws):
    with pytest.raises(ValueError, match="bits_per_value"):
        gz.fixed_rate_compress(np.zeros(4, np.float32), 17)
    blob = gz.fixed_rate_compress(np.arange(10, dtype=np.float32), 4, ws)
    with pytest.raises(gz.DecodeError, match="expected"):
        gz.fixed_rate_decompress(blob[:-1])
    with pytest.raises(gz.DecodeError, match="too short"):
        gz.fixed_rate_decompress(blob[:5])
    with pytest.raises(ValueError, match="offset 3"):
        gz.fixed_rate_compress(np.array([0, 1, 2, np.inf], np.float32), 4, ws)


def test_index_large_reference_blob_and_deep_errors(oracle, ws):
    # a multi-chunk reference blob (payload >> 128 segments of 2 KiB) decoded from host
    # bytes through gz_index, then errors planted deep inside it: the first failing
    # block in walk order is reported, as in codec.py:298-322
    n = 3_000_001
    x = oracle.smooth_field(n) + np.random.default_rng(11).normal(0, 1e-2, n).astype(np.float32)
    ref, offs = oracle.compress(x, 1e-4, threads=8, return_offsets=True)
    assert len(ref) > 24 + 300 * 2048
    y = gz.decompress(ref, ws)
    assert y.tobytes() == oracle.decompress(ref, threads=8).tobytes()
    yh = gz.decompress(torch.frombuffer(bytearray(ref), dtype=torch.uint8).pin_memory(), ws)
    assert yh.numpy().tobytes() == y.tobytes()
    nb = len(offs)
    for k in (nb // 3, nb // 2 + 17, nb - 2):
        bad = bytearray(ref)
        bad[24 + int(offs[k])] = 77
        with pytest.raises(gz.DecodeError, match=f"width code 77 at block {k}"):
            gz.decompress(bytes(bad), ws)
    with pytest.raises(gz.DecodeError, match="truncated"):
        gz.decompress(ref[:-5], ws)
    with pytest.raises(gz.DecodeError, match="trailing"):
        gz.decompress(ref + b"\x00\x00", ws)


@pytest.mark.parametrize("cut_segments", [1, 5, 10, 645])
def test_truncation_exactly_at_a_segment_boundary(cut_segments, oracle, ws):
    # all-zero input -> 5-byte blocks; a payload cut at k * 2048 bytes ends on an index
    # segment boundary with a block ending exactly there: the reference reports the first
    # missing block (codec.py:307-308), never a silent partial decode (gz_index)
    n = 32 * 5 * 2048 * (cut_segments + 1) // 5
    x = np.zeros(n, np.float32)
    blob = oracle.compress(x, 1e-4)
    cut = 24 + 2048 * cut_segments
    nblk = 2048 * cut_segments // 5
    msg = f"truncated payload at block {nblk}"
    with pytest.raises(ValueError, match=msg):
        oracle.decompress(blob[:cut])
    with pytest.raises(gz.DecodeError, match=msg):
        gz.decompress(blob[:cut], ws)
    with pytest.raises(gz.DecodeError, match=msg):
        gz.decompress(torch.frombuffer(bytearray(blob[:cut]), dtype=torch.uint8).cuda(), ws)


@pytest.mark.parametrize("slotted_in", [True, False])
def test_fused_step_reports_nonfinite_local_offset(slotted_in, oracle, ws):
    # every kernel that reads a collective's input records the first non-finite offset of
    # the caller's buffer (codec.py:79-86): the fused step checks `local` (+ report_base),
    # not the received values
    import ctypes
    from paper_2308_05199_b200 import _lib as L
    from paper_2308_05199_b200.comm import _StepIO

    lib = L.lib()
    n = 100_003
    a = oracle.smooth_field(n)
    b = oracle.smooth_field(n, 0.4)
    b[54_321] = np.nan
    b[99_000] = np.inf
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    nt = int(lib.gz_num_tiles(n))
    s = torch.cuda.current_stream().cuda_stream
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))

    def slots():
        sl = torch.empty(int(lib.gz_slots_bytes(n)) + 128, dtype=torch.uint8, device="cuda")
        return sl, (sl.data_ptr() + 127) & ~127, torch.empty(nt, dtype=torch.int32, device="cuda"), \
            torch.empty(32 * nt, dtype=torch.uint8, device="cuda")
    s_in, s_out = slots(), slots()
    io = _StepIO()
    io.out_slots, io.out_sizes, io.out_widths = s_in[1], s_in[2].data_ptr(), s_in[3].data_ptr()
    ws.reset_status()
    L.check(lib.gz_step(ctypes.byref(io), at.data_ptr(), n, 1e-4, 0, None, tws.data_ptr(), tws.numel(),
                        ws.status_ptr(), s), "gz_step")
    assert ws.read_status()[0] == (1 << 64) - 1
    blob = gz.compress(at, 1e-4, ws)
    io2 = _StepIO()
    if slotted_in:
        io2.in_slots, io2.in_sizes, io2.in_widths = s_in[1], s_in[2].data_ptr(), s_in[3].data_ptr()
    else:
        io2.in_blob, io2.in_sidecar = blob.data.data_ptr(), blob.sidecar.data_ptr()
    io2.out_slots, io2.out_sizes, io2.out_widths = s_out[1], s_out[2].data_ptr(), s_out[3].data_ptr()
    io2.report_base = 1000
    acc = torch.empty(n, dtype=torch.float32, device="cuda")
    ws.reset_status()
    L.check(lib.gz_step(ctypes.byref(io2), bt.data_ptr(), n, 1e-4, 0, acc.data_ptr(), tws.data_ptr(), tws.numel(),
                        ws.status_ptr(), s), "gz_step")
    assert int(ws.read_status()[0]) == 1000 + 54_321
