"""Device transports for the reference's collective algorithms (the Transport
seam, /root/reference/pkg/src/gzccl/collectives.py:94-194).

The reference's algorithms (``ring_allreduce_c``, ``binomial_scatter_c``,
``rd_allreduce_c``, ... and ``run_collective``) turn buffers into bytes only
through ``transport.encode(rank, arr) -> (bytes, secs)``,
``transport.decode(rank, blob) -> (arr, secs)`` and
``transport.encode_blocks(rank, blocks) -> (list[bytes], secs)``, and read
``name`` / ``raw_bytes_in`` / ``blob_bytes_out``.  The classes here implement
that protocol with the B200 kernels of ``libgzccl.so``, so a maintainer can
hand them to the reference's own collective code (or install
:func:`make_transport` in place of ``gzccl.collectives.make_transport``)
and get byte-identical messages, outputs and counters.

* :class:`GpuEbCodecTransport` -- the error-bounded codec (EbCodecTransport,
  collectives.py:114-147): encode = gz_compress, decode = gz_index + tile
  decode (any reference blob decodes), encode_blocks = ONE multi-segment
  launch for all blocks (gz_compress_segments, the paper's multi-stream batch).
* :class:`GpuFixedRateTransport` -- the fixed-rate comparator (150-182).
* :class:`RawTransport` -- verbatim float32 payloads (94-111), for the
  lossless twins; no kernels.

``timing``: "model" (default) returns the cost model's seconds
(``params.kernel_time`` / ``multi_launch_time``), exactly as the reference's
transports do, so simulated clocks and counters match the reference run
bit for bit; "measured" returns the device seconds of the kernels (CUDA
events on the launching stream).
"""

from __future__ import annotations

import numpy as np
import torch

from .codec import Workspace, _check_eb, compress, decompress, fixed_rate_compress, fixed_rate_decompress


class _DeviceTransport:
    name = "?"

    def __init__(self, params, *, device=None, timing: str = "model"):
        if timing not in ("model", "measured"):
            raise ValueError(f"timing must be 'model' or 'measured', got {timing!r}")
        if not torch.cuda.is_available():
            raise RuntimeError("device transports need a CUDA device (B200); there is no CPU fallback")
        self.params = params
        self.timing = timing
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.raw_bytes_in = 0
        self.blob_bytes_out = 0
        self._ws: dict[int, Workspace] = {}

    def workspace(self, rank) -> Workspace:
        """One device workspace per rank (simnet.py:82: a workspace per rank)."""
        rid = int(getattr(rank, "id", 0))
        if rid not in self._ws:
            self._ws[rid] = Workspace(self.device)
        return self._ws[rid]

    def _timed(self, fn):
        if self.timing == "model":
            return fn(), None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        return out, e0.elapsed_time(e1) * 1e-3

    def _secs(self, measured, nbytes: int, kind: str) -> float:
        return self.params.kernel_time(nbytes, kind) if measured is None else measured

    def _account(self, rank, raw: int, out: int) -> None:  # collectives.py:124-127
        rank.counters.n_compress += 1
        self.raw_bytes_in += raw
        self.blob_bytes_out += out


def _host_f32(arr) -> np.ndarray:
    return np.ascontiguousarray(arr, dtype="<f4").reshape(-1)


class GpuEbCodecTransport(_DeviceTransport):
    """Error-bounded codec on the B200 (EbCodecTransport, collectives.py:114-147)."""

    name = "ebz"

    def __init__(self, params, eb: float, *, device=None, timing: str = "model"):
        super().__init__(params, device=device, timing=timing)
        self.eb = _check_eb(eb)

    def encode(self, rank, arr) -> tuple[bytes, float]:
        x = _host_f32(arr)
        ws = self.workspace(rank)
        blob, t = self._timed(lambda: compress(x, self.eb, ws))
        self._account(rank, 4 * x.size, len(blob))
        return blob, self._secs(t, 4 * x.size, "compress")

    def decode(self, rank, blob) -> tuple[np.ndarray, float]:
        ws = self.workspace(rank)
        arr, t = self._timed(lambda: decompress(bytes(blob), ws))
        rank.counters.n_decompress += 1
        return arr, self._secs(t, 4 * arr.size, "decompress")

    def encode_blocks(self, rank, blocks) -> tuple[list[bytes], float]:
        """All blocks in ONE multi-segment launch (gz_compress_segments)."""
        from .segments import compress_segments

        blocks = [_host_f32(b) for b in blocks]
        ws = self.workspace(rank)
        counts = [b.size for b in blocks]
        x = torch.from_numpy(np.concatenate(blocks) if blocks else np.empty(0, np.float32)).to(self.device)

        def run():
            seg = compress_segments(x, counts, self.eb, ws)
            packed = seg.packed().cpu().numpy().tobytes()
            out, pos = [], 0
            for s in seg.sizes:
                out.append(packed[pos:pos + s])
                pos += s
            return out

        blobs, t = self._timed(run)
        for b, c in zip(blobs, counts):
            self._account(rank, 4 * c, len(b))
        secs = t if t is not None else self.params.multi_launch_time([4 * c for c in counts], "compress")
        return blobs, secs


class GpuFixedRateTransport(_DeviceTransport):
    """Fixed-rate baseline codec on the B200 (FixedRateTransport, collectives.py:150-182)."""

    name = "fixed-rate"

    def __init__(self, params, bits: int, *, device=None, timing: str = "model"):
        super().__init__(params, device=device, timing=timing)
        self.bits = int(bits)

    def encode(self, rank, arr) -> tuple[bytes, float]:
        x = _host_f32(arr)
        ws = self.workspace(rank)
        blob, t = self._timed(lambda: fixed_rate_compress(x, self.bits, ws))
        self._account(rank, 4 * x.size, len(blob))
        return blob, self._secs(t, 4 * x.size, "compress")

    def decode(self, rank, blob) -> tuple[np.ndarray, float]:
        ws = self.workspace(rank)
        arr, t = self._timed(lambda: fixed_rate_decompress(bytes(blob), ws))
        rank.counters.n_decompress += 1
        return arr, self._secs(t, 4 * arr.size, "decompress")

    def encode_blocks(self, rank, blocks) -> tuple[list[bytes], float]:
        blobs, secs = [], 0.0
        for b in blocks:
            blob, s = self.encode(rank, b)
            blobs.append(blob)
            secs += s
        if self.timing == "model":
            secs = self.params.multi_launch_time([4 * _host_f32(b).size for b in blocks], "compress")
        return blobs, secs


class RawTransport:
    """Verbatim float32 payloads: no kernels, no counters, no loss (collectives.py:94-111)."""

    name = "none"

    def __init__(self, params):
        self.params = params
        self.raw_bytes_in = 0
        self.blob_bytes_out = 0

    def encode(self, rank, arr) -> tuple[bytes, float]:
        return _host_f32(arr).tobytes(), 0.0

    def decode(self, rank, blob) -> tuple[np.ndarray, float]:
        return np.frombuffer(blob, dtype="<f4").copy(), 0.0

    def encode_blocks(self, rank, blocks) -> tuple[list[bytes], float]:
        return [_host_f32(b).tobytes() for b in blocks], 0.0


def make_transport(name: str, params, eb: float | None = None, bits: int = 8, *, timing: str = "model"):
    """make_transport (collectives.py:185-194) returning the device transports."""
    if name == "none":
        return RawTransport(params)
    if name == "ebz":
        if eb is None:
            raise ValueError("the error-bounded codec needs an error bound (eb)")
        return GpuEbCodecTransport(params, eb, timing=timing)
    if name == "fixed-rate":
        return GpuFixedRateTransport(params, bits, timing=timing)
    raise ValueError(f"unknown codec {name!r}, expected 'ebz', 'fixed-rate', or 'none'")
