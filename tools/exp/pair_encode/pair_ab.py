"""A/B of the pair encoder (k_pair_encode) against the one-tile encoder in the same
build: GZ_PAIR_MIN_TILES=1 forces pairs, a huge value disables them.  Prints, per
input, the md5 of (blob, sidecar) and the compress median (us, L2 flushed).

    GZ_PAIR_MIN_TILES=1 python tools/exp/pair_encode/pair_ab.py ; GZ_PAIR_MIN_TILES=999999999 python tools/exp/pair_encode/pair_ab.py
"""
import ctypes
import hashlib
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", "..")))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2308_05199_b200 import _lib  # noqa: E402

L = _lib.lib()
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def inputs():
    rng = np.random.default_rng(5)
    for n in (1000, 4096 * 3 + 17, 1 << 20, (1 << 22) + 999, 1 << 24, 1 << 27):
        yield f"smooth {n}", O.smooth_field(n), 1e-4
    x = O.smooth_field(1 << 22)
    x[rng.integers(0, x.size, 3000)] = rng.standard_normal(3000).astype(np.float32) * 1e4  # raw / wide blocks
    yield "spiky 2^22", x, 1e-4
    y = rng.standard_normal((1 << 22) + 5).astype(np.float32)
    yield "noise 2^22", y, 1e-3
    z = O.smooth_field(1 << 22) * np.float32(1e-38)  # subnormals
    yield "tiny 2^22", z, 1e-45
    yield "eb-edge 2^22", O.smooth_field(1 << 22), 0.5 ** 14


for name, xh, eb in inputs():
    n = xh.size
    x = torch.from_numpy(np.ascontiguousarray(xh, dtype=np.float32)).cuda()
    cap = L.gz_compress_bound(n)
    blob = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    sc = torch.zeros(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
    wsb = L.gz_workspace_bytes(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    L.gz_workspace_init(ws.data_ptr(), wsb, s.cuda_stream)
    st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
    ts = []
    for it in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        rc = L.gz_compress(x.data_ptr(), n, eb, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(), None,
                           ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        assert rc == 0, rc
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    ln = int(st[4].item())
    h = hashlib.md5(blob[:ln].cpu().numpy().tobytes())
    h.update(sc.cpu().numpy().tobytes())
    print(f"{name:16s} eb={eb:<10.3g} len {ln:11d} md5 {h.hexdigest()[:16]}  compress median {ts[len(ts) // 2]:8.1f} us",
          flush=True)
