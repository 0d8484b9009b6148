"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Restates the reference gZCCL codec (``/root/reference/pkg/src/gzccl/codec.py``)
in plain C (``gz_oracle.c``, loaded here through ctypes) and the reference
collective schedules (``collectives.py``) in numpy over that codec.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module; the product package never does.  It is pinned
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``) in ``tests/test_oracle.py``.
"""

from __future__ import annotations

import ctypes
import os
import struct
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgz_oracle.so")

BLOCK = 32
HEADER_BYTES = 24
_SC_HDR = struct.Struct("<QQQ")  # collectives.py:29


class OracleDecodeError(ValueError):
    pass


def build() -> str:
    """Compile the C oracle in place (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i64, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        L.gzo_compress_bound.restype = u64
        L.gzo_compress_bound.argtypes = [u64]
        L.gzo_compress.restype = ctypes.c_int
        L.gzo_compress.argtypes = [p, u64, ctypes.c_double, p, u64, ctypes.POINTER(u64), p, ctypes.POINTER(i64), ctypes.c_int]
        L.gzo_decompress.restype = ctypes.c_int
        L.gzo_decompress.argtypes = [p, u64, p, u64, ctypes.POINTER(u64), ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
        L.gzo_parse_header.restype = ctypes.c_int
        L.gzo_parse_header.argtypes = [p, u64, ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, ctypes.c_int]
        _lib = L
    return _lib


def compress_bound(n: int) -> int:
    return int(lib().gzo_compress_bound(n))


def compress(data, eb: float, threads: int = 1, return_offsets: bool = False):
    """codec.compress (codec.py:149-270) -> bytes [, block offsets (codec.py:241-243)]."""
    x = np.ascontiguousarray(data, dtype="<f4").reshape(-1)
    n = x.size
    cap = compress_bound(n)
    out = np.empty(cap, dtype=np.uint8)
    out_len = ctypes.c_uint64(0)
    bad = ctypes.c_int64(-1)
    nb = -(-n // BLOCK)
    offs = np.empty(max(nb, 1), dtype=np.uint64) if return_offsets else None
    rc = lib().gzo_compress(
        x.ctypes.data, n, float(eb), out.ctypes.data, cap, ctypes.byref(out_len),
        offs.ctypes.data if offs is not None else None, ctypes.byref(bad), int(threads))
    if rc == -1:
        raise ValueError(f"error bound must be positive and finite, got {float(eb)!r}")
    if rc == -2:
        raise ValueError(f"non-finite value at offset {bad.value}")
    if rc != 0:
        raise RuntimeError(f"oracle compress failed rc={rc}")
    blob = out[: out_len.value].tobytes()
    if return_offsets:
        return blob, offs[:nb].astype(np.int64)
    return blob


def decompress(blob, threads: int = 1) -> np.ndarray:
    """codec.decompress (codec.py:284-369)."""
    b = np.frombuffer(bytes(blob), dtype=np.uint8)
    msg = ctypes.create_string_buffer(256)
    n = ctypes.c_uint64(0)
    ebv = ctypes.c_double(0)
    rc = lib().gzo_parse_header(b.ctypes.data, b.size, ctypes.byref(n), ctypes.byref(ebv), msg, 256)
    if rc:
        raise OracleDecodeError(msg.value.decode())
    y = np.empty(max(n.value, 1), dtype=np.float32)
    rc = lib().gzo_decompress(b.ctypes.data, b.size, y.ctypes.data, y.size, ctypes.byref(n), msg, 256, int(threads))
    if rc:
        raise OracleDecodeError(msg.value.decode())
    return y[: n.value].copy()


# ---------------------------------------------------------------------------
# collective schedules (collectives.py), all ranks in one process
# ---------------------------------------------------------------------------


def chunk_spans(n: int, ranks: int):
    """collectives.py:42-45."""
    step = -(-n // ranks) if n else 0
    return [(min(c * step, n), min((c + 1) * step, n)) for c in range(ranks)]


def apply_op(op: str, local: np.ndarray, received: np.ndarray) -> np.ndarray:
    """collectives.py:32-39."""
    if op == "sum":
        return local + received
    if op == "max":
        return np.maximum(local, received)
    raise ValueError(op)


@dataclass
class Trace:
    """(step, src, dst, payload) per message, like Network(record_payloads=True)."""

    msgs: list


def ring_reduce_scatter(bufs, eb, op="sum", trace=None, raw=False, threads=1):
    """ring_reduce_scatter_c, collectives.py:258-291 (two-pass schedule)."""
    enc = (lambda a: np.ascontiguousarray(a, "<f4").tobytes()) if raw else (lambda a: compress(a, eb, threads=threads))
    dec = (lambda b: np.frombuffer(b, "<f4").copy()) if raw else (lambda b: decompress(b, threads=threads))
    bufs = [np.ascontiguousarray(b, "<f4") for b in bufs]
    N = len(bufs)
    n = bufs[0].size
    spans = chunk_spans(n, N)
    acc = [[b[lo:hi].copy() for lo, hi in spans] for b in bufs]
    if N == 1:
        return [bufs[0].copy()]
    for s in range(N - 1):
        sent = []
        for i in range(N):
            blob = enc(acc[i][(i - s) % N])
            sent.append(blob)
            if trace is not None:
                trace.append(("rs", s, i, (i + 1) % N, blob))
        for i in range(N):
            blob = sent[(i - 1) % N]
            c_in = (i - s - 1) % N
            acc[i][c_in] = apply_op(op, acc[i][c_in], dec(blob))
    return [acc[i][(i + 1) % N] for i in range(N)]


def ring_allgather_owned(owned, eb, chunk_of, trace=None, raw=False, threads=1):
    """_ring_allgather, collectives.py:215-244: compress once, forward bytes."""
    enc = (lambda a: np.ascontiguousarray(a, "<f4").tobytes()) if raw else (lambda a: compress(a, eb, threads=threads))
    dec = (lambda b: np.frombuffer(b, "<f4").copy()) if raw else (lambda b: decompress(b, threads=threads))
    N = len(owned)
    gathered = [{chunk_of(i): owned[i]} for i in range(N)]
    if N == 1:
        return gathered
    carry = [enc(owned[i]) for i in range(N)]  # s == 0 encodes once (227)
    for s in range(N - 1):
        if trace is not None:
            for i in range(N):
                trace.append(("ag", s, i, (i + 1) % N, carry[i]))
        new = [carry[(i - 1) % N] for i in range(N)]
        for i in range(N):
            gathered[i][chunk_of((i - 1 - s) % N)] = dec(new[i])
        carry = new
    return gathered


def ring_allreduce(bufs, eb, op="sum", trace=None, raw=False, threads=1):
    """ring_allreduce_c, collectives.py:294-308 (threads: host threads per codec call)."""
    bufs = [np.ascontiguousarray(b, "<f4") for b in bufs]
    N = len(bufs)
    if N == 1:
        return [bufs[0].copy()]
    owned = ring_reduce_scatter(bufs, eb, op, trace, raw, threads)
    gathered = ring_allgather_owned(owned, eb, lambda i: (i + 1) % N, trace, raw, threads)
    return [np.concatenate([gathered[i][c] for c in range(N)]) for i in range(N)]


def ring_allgather(chunks, eb, trace=None, raw=False):
    """ring_allgather_c, collectives.py:247-255."""
    owned = [np.ascontiguousarray(c, "<f4") for c in chunks]
    N = len(owned)
    g = ring_allgather_owned(owned, eb, lambda i: i, trace, raw)
    return [np.concatenate([g[i][c] for c in range(N)]) if N > 1 else owned[i].copy() for i in range(N)]


def cprp2p_allgather(chunks, eb, trace=None):
    """cprp2p_allgather, collectives.py:311-341: every hop decompresses and
    re-compresses what it forwards."""
    owned = [np.ascontiguousarray(c, "<f4") for c in chunks]
    N = len(owned)
    if N == 1:
        return [owned[0].copy()]
    gathered = [{i: owned[i]} for i in range(N)]
    current = list(owned)
    for s in range(N - 1):
        sent = [compress(current[i], eb) for i in range(N)]
        if trace is not None:
            for i in range(N):
                trace.append(("cp", s, i, (i + 1) % N, sent[i]))
        for i in range(N):
            vals = decompress(sent[(i - 1) % N])
            gathered[i][(i - 1 - s) % N] = vals
            current[i] = vals
    return [np.concatenate([gathered[i][c] for c in range(N)]) for i in range(N)]


def rd_plan(N: int):
    """RecursiveDoublingPlan, collectives.py:48-86: (pof2, r, steps, role, remapped, actual)."""
    pof2 = 1 << (N.bit_length() - 1)
    r = N - pof2
    steps = pof2.bit_length() - 1

    def role(i):
        return ("donor" if i % 2 == 0 else "absorber") if i < 2 * r else "direct"

    def remapped(i):
        return i // 2 if role(i) == "absorber" else i - r

    def actual(v):
        return 2 * v + 1 if v < r else v + r

    return pof2, r, steps, role, remapped, actual


def rd_allreduce(bufs, eb, op="sum", trace=None, raw=False):
    """rd_allreduce_c, collectives.py:349-424: donors fold into absorbers,
    log2(pof2) whole-buffer exchanges (each side keeps op(own, decoded
    partner)), absorbers send the result back compressed."""
    enc = (lambda a: np.ascontiguousarray(a, "<f4").tobytes()) if raw else (lambda a: compress(a, eb))
    dec = (lambda b: np.frombuffer(b, "<f4").copy()) if raw else decompress
    data = [np.ascontiguousarray(b, "<f4").copy() for b in bufs]
    N = len(data)
    if N == 1:
        return [data[0].copy()]
    pof2, r, steps, role, remapped, actual = rd_plan(N)
    donors = [i for i in range(N) if role(i) == "donor"]
    parts = [i for i in range(N) if role(i) != "donor"]
    if r:
        sent = {}
        for i in donors:  # 381-386
            sent[i] = enc(data[i])
            if trace is not None:
                trace.append(("rd", -1, i, i + 1, sent[i]))
        for i in range(N):  # 389-397
            if role(i) == "absorber":
                data[i] = apply_op(op, data[i], dec(sent[i - 1]))
    for t in range(steps):  # 399-418
        sent = {}
        for i in parts:
            partner = actual(remapped(i) ^ (1 << t))
            sent[i] = enc(data[i])
            if trace is not None:
                trace.append(("rd", t, i, partner, sent[i]))
        for i in parts:
            partner = actual(remapped(i) ^ (1 << t))
            data[i] = apply_op(op, data[i], dec(sent[partner]))
    if r:
        sent = {}
        for i in range(N):  # 420-427
            if role(i) == "absorber":
                sent[i] = enc(data[i])
                if trace is not None:
                    trace.append(("rd", steps, i, i - 1, sent[i]))
        for i in donors:  # 430-435
            data[i] = dec(sent[i + 1])
    return data


def scatter_children(vr: int, size: int):
    """_scatter_children, collectives.py:449-464."""
    mask = 1
    while mask < size:
        if vr & mask:
            break
        mask <<= 1
    extent = mask
    sends = []
    mask >>= 1
    while mask:
        child = vr + mask
        if child < size:
            sends.append((child, child, min(child + mask, size)))
        mask >>= 1
    return extent, sends


def pack_scatter_msg(sizes, lo, hi, frag: bytes) -> bytes:
    """_pack_scatter_msg, collectives.py:432-434."""
    return _SC_HDR.pack(len(sizes), lo, hi) + np.asarray(sizes, dtype="<u8").tobytes() + frag


def binomial_scatter(data, N, eb, root=0, counts=None, trace=None, threads=1):
    """binomial_scatter_c, collectives.py:467-532 (messages appended to trace;
    threads: host threads per codec call)."""
    data = np.ascontiguousarray(data, "<f4").reshape(-1)
    if counts is None:
        counts = [hi - lo for lo, hi in chunk_spans(data.size, N)]
    counts = [int(c) for c in counts]
    if len(counts) != N or any(c < 0 for c in counts) or sum(counts) != data.size:
        raise ValueError("bad counts")
    rank_lo = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    slices = [data[rank_lo[i] : rank_lo[i + 1]] for i in range(N)]
    outputs = [None] * N
    outputs[root] = slices[root].copy()
    if N == 1:
        return outputs
    order = [(root + j) % N for j in range(N)]
    blobs = [compress(slices[r], eb, threads=threads) for r in order]
    sizes = [len(b) for b in blobs]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    payload = b"".join(blobs)
    inbox = {}
    _, root_sends = scatter_children(0, N)
    for child, lo, hi in root_sends:
        msg = pack_scatter_msg(sizes, lo, hi, payload[offs[lo] : offs[hi - 1] + sizes[hi - 1]])
        inbox[order[child]] = msg
        if trace is not None:
            trace.append((root, order[child], msg))
    for vr in range(1, N):
        me = order[vr]
        _, sends = scatter_children(vr, N)
        msg = inbox[me]
        cnt, lo, hi = _SC_HDR.unpack_from(msg)
        frag = msg[_SC_HDR.size + 8 * cnt :]
        for child, clo, chi in sends:
            sub = frag[offs[clo] - offs[lo] : offs[chi - 1] + sizes[chi - 1] - offs[lo]]
            cmsg = pack_scatter_msg(sizes, clo, chi, sub)
            inbox[order[child]] = cmsg
            if trace is not None:
                trace.append((me, order[child], cmsg))
        own = frag[offs[vr] - offs[lo] : offs[vr] + sizes[vr] - offs[lo]]
        outputs[me] = decompress(own, threads=threads)
    return outputs


def smooth_field(n: int, phase: float = 0.0) -> np.ndarray:
    """SURVEY §8(d) cfg1/cfg2 field: f32(0.5 sin(2πi/65536 + φ) + 0.25 sin(2πi/4099 + φ))."""
    i = np.arange(n, dtype=np.float64)
    return (0.5 * np.sin(2 * np.pi * i / 65536 + phase) + 0.25 * np.sin(2 * np.pi * i / 4099 + phase)).astype(np.float32)


# ---------------------------------------------------------------------------
# fixed-rate baseline codec (codec.py:442-489), numpy restatement
# ---------------------------------------------------------------------------
FR_HEADER_BYTES = 17  # struct "<QBff": n, bits, lo, hi


def np_extremum_avx512(x: np.ndarray, op: str) -> float:
    """x.min() / x.max() of a contiguous float32 array exactly as numpy 2.x
    computes it on an AVX-512 host (the host the reference's goldens were made
    on), INCLUDING the sign of a zero result, which numpy's SIMD reduction
    makes order-dependent (codec.py:454-455 calls x.min() / x.max()):
    numpy's simd_reduce_c (loops_minmax.dispatch.c.src) starts 16 lanes at
    x[0], folds x[1 + 16j + l] into lane l with vminps / vmaxps (a tie returns
    the SECOND operand), combines the lanes with GCC's _mm512_reduce_min_ps /
    _mm512_reduce_max_ps tree and folds the (n-1) % 16 tail values in one by
    one (ties again return the later value).  Pure Python, for small inputs."""
    x = np.ascontiguousarray(x, "<f4").reshape(-1)
    better = (lambda a, b: a < b) if op == "min" else (lambda a, b: a > b)

    def f(a, b):  # (value, index); the first operand only wins a strict comparison
        return a if better(a[0], b[0]) else b

    n = x.size
    nv = (n - 1) // 16
    lane = [(float(x[0]), 0)] * 16
    for j in range(nv):
        for l in range(16):
            i = 1 + 16 * j + l
            lane[l] = f(lane[l], (float(x[i]), i))
    t3 = [f(lane[8 + i], lane[i]) for i in range(8)]
    t6 = [f(t3[4 + i], t3[i]) for i in range(4)]
    r = f(f(t6[0], t6[2]), f(t6[1], t6[3]))
    for i in range(1 + 16 * nv, n):
        r = f(r, (float(x[i]), i))
    return float(x[r[1]])


def fixed_rate_compress(data, bits_per_value: int) -> bytes:
    import struct

    x = np.ascontiguousarray(data, "<f4").reshape(-1)
    b = int(bits_per_value)
    if not 1 <= b <= 16:
        raise ValueError(f"bits_per_value must be in [1, 16], got {b}")
    n = x.size
    lo = float(x.min()) if n else 0.0
    hi = float(x.max()) if n else 0.0
    # a zero extremum's sign is order-dependent in numpy: follow the AVX-512 reduction
    if n and lo == 0.0:
        lo = np_extremum_avx512(x, "min") if n < 100_000 else _zero_sign_fast(x, lo)
    if n and hi == 0.0:
        hi = np_extremum_avx512(x, "max") if n < 100_000 else _zero_sign_fast(x, hi)
    head = struct.pack("<QBff", n, b, lo, hi)
    if n == 0:
        return head
    levels = (1 << b) - 1
    if hi > lo:
        v = (x.astype(np.float64) - lo) / (hi - lo) * levels
        q = np.floor(np.abs(v) + 0.5) * np.sign(v)
        q = np.clip(q, 0, levels).astype(np.uint32)
    else:
        q = np.zeros(n, dtype=np.uint32)
    bitsarr = ((q[:, None] >> np.arange(b, dtype=np.uint32)[None, :]) & 1).astype(np.uint8).reshape(-1)
    return head + np.packbits(bitsarr, bitorder="little").tobytes()


def _zero_sign_fast(x: np.ndarray, v: float) -> float:
    """np_extremum_avx512 for a zero extremum on large inputs (vectorised):
    the winner is the last zero of the scalar tail, else the lane the GCC
    reduction tree selects among the lanes whose last zero exists."""
    n = x.size
    nv = (n - 1) // 16
    tail = np.flatnonzero(x[1 + 16 * nv:] == 0.0)
    if tail.size:
        return float(x[1 + 16 * nv + tail[-1]])
    last = [-1] * 16
    if nv:
        body = x[1:1 + 16 * nv].reshape(nv, 16) == 0.0
        for l in range(16):
            z = np.flatnonzero(body[:, l])
            if z.size:
                last[l] = 1 + 16 * int(z[-1]) + l
    x0z = x[0] == 0.0
    lane = [last[l] if last[l] >= 0 else (0 if x0z else -1) for l in range(16)]

    def f(a, b):
        return b if b >= 0 else a

    t3 = [f(lane[8 + i], lane[i]) for i in range(8)]
    t6 = [f(t3[4 + i], t3[i]) for i in range(4)]
    r = f(f(t6[0], t6[2]), f(t6[1], t6[3]))
    return float(x[r]) if r >= 0 else v


def fixed_rate_decompress(blob) -> np.ndarray:
    import struct

    blob = bytes(blob)
    if len(blob) < FR_HEADER_BYTES:
        raise ValueError(f"blob too short for fixed-rate header ({len(blob)} bytes)")
    n, b, lo, hi = struct.unpack_from("<QBff", blob)
    if not 1 <= b <= 16:
        raise ValueError(f"invalid bits_per_value {b} in header")
    expect = (n * b + 7) // 8
    payload = np.frombuffer(blob, dtype=np.uint8, offset=FR_HEADER_BYTES)
    if payload.size != expect:
        raise ValueError(f"payload is {payload.size} bytes, expected {expect}")
    if n == 0:
        return np.empty(0, dtype=np.float32)
    bitsarr = np.unpackbits(payload, bitorder="little")[: n * b].reshape(n, b).astype(np.uint32)
    q = (bitsarr << np.arange(b, dtype=np.uint32)[None, :]).sum(axis=1)
    levels = (1 << b) - 1
    if hi > lo:
        vals = lo + q.astype(np.float64) * ((hi - lo) / levels)
    else:
        vals = np.full(n, lo, dtype=np.float64)
    return vals.astype(np.float32)
