"""Error-bounded codec with the reference's frozen byte format, on B200.

Host-side mirror of ``gzccl.codec`` (/root/reference/pkg/src/gzccl/codec.py):
same names, arguments, return kinds and error types/messages.  All arithmetic
runs in the sm_100a kernels of ``libgzccl.so`` (csrc/gz_codec.cu); this module
only validates arguments, manages device buffers and raises errors.

Inputs may be numpy arrays / array-likes / bytes (the reference's kinds: the
result is ``bytes`` / ``np.ndarray``) or CUDA tensors (the result stays on the
device: :class:`DeviceBlob` / ``torch.Tensor``).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

MAGIC = b"GZC1"                      # codec.py:41
BLOCK = 32                           # codec.py:42
HEADER = struct.Struct("<4s4xQd")    # codec.py:43
HEADER_BYTES = HEADER.size           # codec.py:44
RAW_WIDTH = 255                      # codec.py:45
MAX_STEP = 1 << 30                   # codec.py:46
_NONE = (1 << 64) - 1


class DecodeError(ValueError):
    """Raised for malformed, truncated, or inconsistent compressed bytes (codec.py:52-53)."""


def _check_eb(eb) -> float:  # codec.py:89-93
    eb = float(eb)
    if not (math.isfinite(eb) and eb > 0.0):
        raise ValueError(f"error bound must be positive and finite, got {eb!r}")
    return eb


def _check_block(block) -> None:
    if int(block) != BLOCK:
        raise ValueError(f"block size must be {BLOCK}: the byte format is frozen (codec.py:42-43)")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _device_of(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2308_05199_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


class Workspace:
    """Reusable device scratch keyed by role (codec.py:56-76).

    Holds the look-back tile workspace (zeroed once, then self-resetting),
    the status/length record, and role-keyed byte buffers that grow by 1.25x.
    Not thread-safe: one workspace per concurrent caller / stream.
    """

    def __init__(self, device=None):
        self.device = _device_of(device)
        self._store: dict[str, torch.Tensor] = {}
        self._tile: torch.Tensor | None = None
        # [0..3] gz_status, [4] compressed length, [5..7] spare
        self.status = torch.empty(8, dtype=torch.int64, device=self.device)
        self._host = torch.empty(8, dtype=torch.int64, pin_memory=True)

    def get(self, key: str, nbytes: int) -> torch.Tensor:
        buf = self._store.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes + (nbytes >> 2), 64), dtype=torch.uint8, device=self.device)
            self._store[key] = buf
        return buf[:nbytes]

    def tile_ws(self, nbytes: int) -> torch.Tensor:
        if self._tile is None or self._tile.numel() < nbytes:
            nbytes = max(nbytes + (nbytes >> 2), 4096)
            self._tile = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            L.check(L.lib().gz_workspace_init(self._tile.data_ptr(), nbytes, _stream()), "gz_workspace_init")
        return self._tile

    # status helpers -------------------------------------------------------
    def status_ptr(self) -> int:
        return self.status.data_ptr()

    def len_ptr(self) -> int:
        return self.status.data_ptr() + 32

    def reset_status(self, stream=None) -> None:
        L.check(L.lib().gz_status_reset(self.status_ptr(), _stream(stream)), "gz_status_reset")

    def read_status(self, stream=None) -> np.ndarray:
        """Synchronise the stream and return the 8-word status record."""
        self._host.copy_(self.status, non_blocking=True)
        (stream or torch.cuda.current_stream()).synchronize()
        return self._host.numpy().view(np.uint64).copy()


_default_ws: dict[int, Workspace] = {}


def _ws_for(workspace, device) -> Workspace:
    if workspace is not None:
        return workspace
    key = device.index
    if key not in _default_ws:
        _default_ws[key] = Workspace(device)
    return _default_ws[key]


@dataclass
class DeviceBlob:
    """A compressed blob resident in device memory.

    ``data`` holds exactly the reference bytes (header included); ``sidecar``
    holds the tile/group offsets the device decoder uses to find blocks
    without the sequential walk.  ``bytes(blob)`` is the reference blob.
    """

    data: torch.Tensor
    sidecar: torch.Tensor
    n: int
    eb: float
    block_offsets: torch.Tensor | None = None

    def __len__(self) -> int:
        return int(self.data.numel())

    def __bytes__(self) -> bytes:
        return self.data.cpu().numpy().tobytes()

    def tobytes(self) -> bytes:
        return bytes(self)


def _as_device_f32(data, device=None) -> tuple[torch.Tensor, bool]:
    """codec._ingest (codec.py:79-86) minus the finiteness scan, which runs on the device."""
    if isinstance(data, torch.Tensor) and data.is_cuda:
        if data.dim() != 1:
            raise ValueError("expected a flat 1-D sequence of binary32 values")
        return data.detach().to(torch.float32).contiguous(), True
    if isinstance(data, torch.Tensor):  # host tensor (ideally pinned): async H2D
        if data.dim() != 1:
            raise ValueError("expected a flat 1-D sequence of binary32 values")
        dev = _device_of(device)
        return data.detach().to(torch.float32).contiguous().to(dev, non_blocking=True), False
    x = np.ascontiguousarray(data, dtype="<f4")
    if x.ndim != 1:
        raise ValueError("expected a flat 1-D sequence of binary32 values")
    dev = _device_of(device)
    return torch.from_numpy(x).to(dev, non_blocking=False), False


def _on(stream):
    """Run a call's copies and kernels on ``stream`` (default: the current stream)."""
    import contextlib

    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def compress(data, eb, workspace: Workspace | None = None, *, block: int = BLOCK, return_offsets: bool = False,
             stream=None):
    """Compress binary32 values under an absolute error bound (codec.py:149-270).

    Host input -> ``bytes`` (byte-identical to the reference).  CUDA tensor
    input -> :class:`DeviceBlob`.  Host torch tensor (pinned) -> pinned host
    uint8 tensor holding the reference bytes.  Rejects non-finite input (``ValueError``
    naming the first bad offset) and non-positive bounds.  Every copy and
    kernel of the call is ordered on ``stream``: calls on distinct streams with
    distinct workspaces run concurrently (e.g. one host buffer's H2D beside
    another's D2H).
    """
    with _on(stream):
        return _compress(data, eb, workspace, block, return_offsets, stream)


def _compress(data, eb, workspace, block, return_offsets, stream):
    _check_block(block)
    ebf = _check_eb(eb)
    x, on_dev = _as_device_f32(data, workspace.device if workspace is not None else None)
    ws = _ws_for(workspace, x.device)
    lib = L.lib()
    n = x.numel()
    nb = -(-n // BLOCK)
    cap = int(lib.gz_compress_bound(n))
    blob = torch.empty(cap, dtype=torch.uint8, device=x.device)
    sidecar = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device=x.device)
    offs = torch.empty(max(nb, 1), dtype=torch.int64, device=x.device) if return_offsets else None
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    s = _stream(stream)
    ws.reset_status(stream)
    L.check(lib.gz_compress(x.data_ptr(), n, ebf, BLOCK, blob.data_ptr(), cap, ws.len_ptr(), sidecar.data_ptr(),
                            _ptr(offs), tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_compress")
    st = ws.read_status(stream)
    if st[0] != _NONE:
        raise ValueError(f"non-finite value at offset {int(st[0])}")
    length = int(st[4])
    db = DeviceBlob(blob[:length], sidecar, n, ebf, offs[:nb] if offs is not None else None)
    if on_dev:
        return db
    if isinstance(data, torch.Tensor):  # host tensor in -> pinned host uint8 tensor out
        host = torch.empty(length, dtype=torch.uint8, pin_memory=True)
        host.copy_(blob[:length], non_blocking=True)
        (stream or torch.cuda.current_stream()).synchronize()
        return host
    out = bytes(db)
    if return_offsets:
        return out, offs[:nb].cpu().numpy()
    return out


def _parse_header(blob: bytes) -> tuple[int, float]:  # codec.py:273-281
    if len(blob) < HEADER_BYTES:
        raise DecodeError(f"blob too short for header ({len(blob)} bytes)")
    magic, n, eb = HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise DecodeError(f"bad magic {magic!r}")
    if not (math.isfinite(eb) and eb > 0.0):
        raise DecodeError(f"invalid error bound in header: {eb!r}")
    return n, eb


def _raise_decode(st: np.ndarray, n: int) -> None:
    e = int(st[1])
    if e == _NONE:
        return
    code = e & 0xFF
    w = (e >> 8) & 0xFFFF
    blk = e >> 24
    if code == 1:
        raise DecodeError(f"unknown width code {w} at block {blk}")
    if code == 2:
        raise DecodeError(f"truncated payload at block {blk}")
    if code == 3:
        raise DecodeError(f"{int(st[2])} trailing bytes after last block")
    raise DecodeError(f"inconsistent compressed stream at block {blk} (code {code})")


def _decode_with_sidecar(blob_dev: torch.Tensor, sidecar: torch.Tensor, n: int, eb: float, ws: Workspace, stream,
                         check: bool) -> torch.Tensor:
    y = torch.empty(n, dtype=torch.float32, device=blob_dev.device)
    if n == 0:
        return y
    if check:
        ws.reset_status(stream)
    L.check(L.lib().gz_decompress_sidecar(blob_dev.data_ptr(), sidecar.data_ptr(), n, eb, y.data_ptr(),
                                          ws.status_ptr(), _stream(stream)), "gz_decompress_sidecar")
    if check:
        _raise_decode(ws.read_status(stream), n)
    return y


def build_sidecar(blob_dev: torch.Tensor, n: int, payload_len: int, ws: Workspace, stream=None) -> torch.Tensor:
    """Build the device sidecar of a reference blob, validating it like codec.py:298-322."""
    lib = L.lib()
    sidecar = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device=blob_dev.device)
    iws = ws.get("index.ws", int(lib.gz_index_workspace_bytes(payload_len)))
    ws.reset_status(stream)
    L.check(lib.gz_index(blob_dev.data_ptr(), payload_len, n, sidecar.data_ptr(), iws.data_ptr(), iws.numel(),
                         ws.status_ptr(), _stream(stream)), "gz_index")
    _raise_decode(ws.read_status(stream), n)
    return sidecar


def decompress(blob, workspace: Workspace | None = None, *, stream=None, check: bool = True):
    """Decode a compressed blob back to float32 values (codec.py:284-369).

    ``bytes``-like input -> ``np.ndarray``; :class:`DeviceBlob` or CUDA uint8
    tensor -> ``torch.Tensor`` on that device; host uint8 tensor -> pinned
    host float32 tensor.  Raises :class:`DecodeError` on
    malformed headers, truncated payloads or unknown width codes.  Ordered on
    ``stream`` like :func:`compress`.
    """
    with _on(stream):
        return _decompress(blob, workspace, stream, check)


def _decompress(blob, workspace, stream, check):
    if isinstance(blob, DeviceBlob):
        ws = _ws_for(workspace, blob.data.device)
        return _decode_with_sidecar(blob.data, blob.sidecar, blob.n, blob.eb, ws, stream, check)
    if isinstance(blob, torch.Tensor) and not blob.is_cuda:  # host uint8 tensor (ideally pinned)
        hb = blob.reshape(-1)
        total = int(hb.numel())
        n, eb = _parse_header(hb[:HEADER_BYTES].numpy().tobytes())
        if n == 0:
            if total > HEADER_BYTES:
                raise DecodeError("trailing bytes after empty payload")
            return torch.empty(0, dtype=torch.float32)
        dev = _device_of(workspace.device if workspace is not None else None)
        ws = _ws_for(workspace, dev)
        buf = ws.get("decompress.blob", total + 64)
        buf[:total].copy_(hb, non_blocking=True)
        sidecar = build_sidecar(buf, n, total - HEADER_BYTES, ws, stream)
        y = _decode_with_sidecar(buf, sidecar, n, eb, ws, stream, check)
        out = torch.empty(n, dtype=torch.float32, pin_memory=True)
        out.copy_(y, non_blocking=True)
        (stream or torch.cuda.current_stream()).synchronize()
        return out
    on_dev = isinstance(blob, torch.Tensor) and blob.is_cuda
    if on_dev:
        head = bytes(blob[:HEADER_BYTES].cpu().numpy().tobytes())
        total = int(blob.numel())
        n, eb = _parse_header(head if total >= HEADER_BYTES else bytes(blob.cpu().numpy().tobytes()))
        dev = blob.device
        src = blob
    else:
        raw = bytes(blob)
        n, eb = _parse_header(raw)
        total = len(raw)
        dev = _device_of(workspace.device if workspace is not None else None)
        src = None
    payload_len = total - HEADER_BYTES
    if n == 0:  # codec.py:293-296
        if payload_len:
            raise DecodeError("trailing bytes after empty payload")
        return torch.empty(0, dtype=torch.float32, device=dev) if on_dev else np.empty(0, dtype=np.float32)
    ws = _ws_for(workspace, dev)
    # device copy with read slack (the decoder stages 16-byte chunks)
    buf = torch.zeros(total + 64, dtype=torch.uint8, device=dev)
    if on_dev:
        buf[:total].copy_(src.reshape(-1))
    else:
        buf[:total].copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    sidecar = build_sidecar(buf, n, payload_len, ws, stream)
    y = _decode_with_sidecar(buf, sidecar, n, eb, ws, stream, check)
    return y if on_dev else y.cpu().numpy()


# ---------------------------------------------------------------------------
# per-segment blobs (codec.py:372-439)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BlockTable:
    """Per-block compressed sizes and starting offsets into a packed payload (codec.py:372-405)."""

    sizes: tuple[int, ...]
    offsets: tuple[int, ...] = field(default=())

    def __post_init__(self):
        if not self.offsets:
            object.__setattr__(self, "offsets", self._offsets_from(self.sizes))
        if len(self.offsets) != len(self.sizes):
            raise ValueError("sizes and offsets length mismatch")
        if self.sizes:
            if self.offsets[0] != 0:
                raise ValueError("first offset must be 0")
            for i in range(len(self.sizes) - 1):
                if self.offsets[i + 1] != self.offsets[i] + self.sizes[i]:
                    raise ValueError(f"offset chain broken at block {i}")

    @staticmethod
    def _offsets_from(sizes) -> tuple[int, ...]:
        offs, acc = [], 0
        for s in sizes:
            offs.append(acc)
            acc += s
        return tuple(offs)

    @property
    def count(self) -> int:
        return len(self.sizes)

    @property
    def total_bytes(self) -> int:
        return sum(self.sizes)


def compress_blocks(data, counts, eb, workspace: Workspace | None = None):
    """Independently compress consecutive blocks of ``counts[i]`` values (codec.py:408-427).

    All blocks are encoded by one multi-segment launch (csrc gz_compress_segments,
    the paper's multi-stream compression).
    """
    from .segments import compress_segments

    x, on_dev = _as_device_f32(data, workspace.device if workspace is not None else None)
    counts = [int(c) for c in counts]
    if any(c < 0 for c in counts):
        raise ValueError("block counts must be non-negative")
    if sum(counts) != x.numel():
        raise ValueError(f"block counts sum to {sum(counts)}, buffer has {x.numel()} values")
    ebf = _check_eb(eb)
    ws = _ws_for(workspace, x.device)
    seg = compress_segments(x, counts, ebf, ws)
    table = BlockTable(sizes=tuple(seg.sizes))
    if on_dev:
        return seg, table
    return seg.packed_bytes(), table


def decompress_block(payload, table: BlockTable, index: int, workspace: Workspace | None = None):
    """Decode one block of a packed payload, touching only that block's bytes (codec.py:430-439)."""
    if not 0 <= index < table.count:
        raise IndexError(f"block index {index} out of range [0, {table.count})")
    off = table.offsets[index]
    end = off + table.sizes[index]
    if isinstance(payload, torch.Tensor) and payload.is_cuda:
        if end > payload.numel():
            raise DecodeError(f"payload shorter than block {index} extent")
        return decompress(payload[off:end], workspace)
    payload = bytes(payload)
    if end > len(payload):
        raise DecodeError(f"payload shorter than block {index} extent")
    return decompress(payload[off:end], workspace)


FR_HEADER = struct.Struct("<QBff")  # codec.py:48
FR_HEADER_BYTES = FR_HEADER.size  # 17


def fixed_rate_compress(data, bits_per_value: int, workspace: Workspace | None = None, stream=None):
    """Fixed-rate baseline (codec.py:442-468): uniform quantisation over
    [min, max] to ``bits_per_value`` bits, ``17 + ceil(n*b/8)`` bytes.  Host
    input -> ``bytes`` (byte-identical to the reference); CUDA tensor -> a
    CUDA uint8 tensor holding the same bytes."""
    b = int(bits_per_value)
    if not 1 <= b <= 16:
        raise ValueError(f"bits_per_value must be in [1, 16], got {b}")
    x, on_dev = _as_device_f32(data, workspace.device if workspace is not None else None)
    ws = _ws_for(workspace, x.device)
    n = x.numel()
    lib = L.lib()
    cap = int(lib.gz_fr_bound(n, b))
    out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    scratch = ws.get("fixed_rate.scratch", int(lib.gz_fr_workspace_bytes()))
    ws.reset_status(stream)
    L.check(lib.gz_fr_compress(x.data_ptr(), n, b, out.data_ptr(), cap, ws.len_ptr(), scratch.data_ptr(),
                               ws.status_ptr(), _stream(stream)), "gz_fr_compress")
    st = ws.read_status(stream)
    if st[0] != _NONE:
        raise ValueError(f"non-finite value at offset {int(st[0])}")  # codec.py:83-85
    blob = out[: int(st[4])]
    return blob if on_dev else blob.cpu().numpy().tobytes()


def fixed_rate_decompress(blob, workspace: Workspace | None = None, stream=None):
    """Inverse of :func:`fixed_rate_compress` (codec.py:471-489), same errors."""
    if isinstance(blob, torch.Tensor) and blob.is_cuda:
        dev_blob, host_head = blob, blob[:FR_HEADER_BYTES].cpu().numpy().tobytes()
        total = blob.numel()
    else:
        raw = bytes(blob)
        dev_blob, host_head, total = None, raw[:FR_HEADER_BYTES], len(raw)
    if len(host_head) < FR_HEADER_BYTES:
        raise DecodeError(f"blob too short for fixed-rate header ({len(host_head)} bytes)")
    n, b, lo, hi = FR_HEADER.unpack_from(host_head)
    if not 1 <= b <= 16:
        raise DecodeError(f"invalid bits_per_value {b} in header")
    expect = (n * b + 7) // 8
    if total - FR_HEADER_BYTES != expect:
        raise DecodeError(f"payload is {total - FR_HEADER_BYTES} bytes, expected {expect}")
    dev = _device_of(workspace.device if workspace is not None else (dev_blob.device if dev_blob is not None else None))
    if dev_blob is None:
        dev_blob = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    L.check(L.lib().gz_fr_decompress(dev_blob.data_ptr(), n, b, y.data_ptr(), _stream(stream)), "gz_fr_decompress")
    if isinstance(blob, torch.Tensor) and blob.is_cuda:
        return y
    return y.cpu().numpy()


def worst_case_blob_bytes(n: int) -> int:
    """Upper bound on compressed size: header plus all-raw blocks (codec.py:492-494)."""
    return HEADER_BYTES + -(-n // BLOCK) * (1 + 4 + 4 * BLOCK)


def compressed_bound(n: int) -> int:
    """Device buffer bound used by this package (129 B per raw block + read slack)."""
    return int(L.lib().gz_compress_bound(n))
