"""Multi-segment compression: N independent blobs in one launch.

Device form of ``codec.compress_blocks`` (codec.py:408-427) used by the
binomial scatter root (collectives.py:497): the paper's multi-stream batch
 becomes one kernel whose CTAs are spread over segments.
Each blob lands in its own worst-case-sized slot; lengths stay on the device
until a caller needs them on the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .codec import BLOCK, DeviceBlob, Workspace, _NONE, _stream


def _align16(v: int) -> int:
    return (v + 15) & ~15


@dataclass
class SegmentBlobs:
    payload: torch.Tensor        # uint8, slot i at slot_off[i]
    slot_off: list
    sidecars: torch.Tensor       # uint8, sidecar i at sidecar_off[i]
    sidecar_off: list
    d_lens: torch.Tensor         # int64[nseg] blob lengths (device)
    counts: list
    eb: float
    _lens: list | None = None

    @property
    def sizes(self) -> list:
        if self._lens is None:
            self._lens = [int(v) for v in self.d_lens.cpu().tolist()]
        return self._lens

    def blob(self, i: int) -> DeviceBlob:
        o = self.slot_off[i]
        sc = self.sidecar_off[i]
        nsc = int(L.lib().gz_sidecar_bytes(self.counts[i]))
        return DeviceBlob(self.payload[o : o + self.sizes[i]], self.sidecars[sc : sc + nsc], self.counts[i], self.eb)

    def packed(self) -> torch.Tensor:
        """Blobs concatenated in order (the reference's packed payload), on the device."""
        sizes = self.sizes
        out = torch.empty(sum(sizes), dtype=torch.uint8, device=self.payload.device)
        pos = 0
        for i, s in enumerate(sizes):
            out[pos : pos + s].copy_(self.payload[self.slot_off[i] : self.slot_off[i] + s])
            pos += s
        return out

    def packed_bytes(self) -> bytes:
        return self.packed().cpu().numpy().tobytes()


def compress_segments(x: torch.Tensor, counts, eb: float, ws: Workspace, stream=None, check: bool = True) -> SegmentBlobs:
    lib = L.lib()
    counts = [int(c) for c in counts]
    nseg = len(counts)
    slot_off, sc_off = [], []
    pos = sc = 0
    for c in counts:
        slot_off.append(pos)
        sc_off.append(sc)
        pos += _align16(int(lib.gz_compress_bound(c)))
        sc += _align16(int(lib.gz_sidecar_bytes(c)))
    dev = x.device
    payload = torch.empty(max(pos, 16), dtype=torch.uint8, device=dev)
    sidecars = torch.empty(max(sc, 16), dtype=torch.uint8, device=dev)
    d_lens = torch.empty(max(nseg, 1), dtype=torch.int64, device=dev)
    arr = ctypes.c_uint64 * max(nseg, 1)
    h_counts, h_slot, h_sc = arr(*counts), arr(*slot_off), arr(*sc_off)
    tws = ws.tile_ws(int(lib.gz_segments_workspace_bytes(h_counts, nseg)))
    if check:
        ws.reset_status(stream)
    L.check(lib.gz_compress_segments(x.data_ptr(), h_counts, nseg, float(eb), payload.data_ptr(), h_slot,
                                     d_lens.data_ptr(), sidecars.data_ptr(), h_sc, None, tws.data_ptr(), tws.numel(),
                                     ws.status_ptr(), _stream(stream)), "gz_compress_segments")
    if check:
        st = ws.read_status(stream)
        if st[0] != _NONE:
            raise ValueError(f"non-finite value at offset {int(st[0])}")
    return SegmentBlobs(payload, slot_off, sidecars, sc_off, d_lens[:nseg], counts, float(eb))
