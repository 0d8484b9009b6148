"""Codec kernels with local vs peer (NVLink) operands, one process, 2 GPUs.
python tools/prof_peer.py [log2 n]"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch

import paper_2308_05199_b200._lib as _L0
if os.environ.get("GZ_LIB"): _L0.LIB_PATH = os.environ["GZ_LIB"]
import paper_2308_05199_b200 as gz
from oracle import oracle as O
from paper_2308_05199_b200 import _lib as L

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 25)
eb = 1e-4
lib = L.lib()
torch.cuda.set_device(0)
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
L.check(lib.gz_enable_peer_access(1), "peer")
x = torch.from_numpy(O.smooth_field(n, 0.0)).to(d0)
y = torch.from_numpy(O.smooth_field(n, 0.37)).to(d0)
ws = gz.Workspace(d0)
cap = int(lib.gz_compress_bound(n))
scb = int(lib.gz_sidecar_bytes(n))
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=d0)
s = torch.cuda.current_stream(d0).cuda_stream


def bufs(dev):
    return (torch.empty(cap, dtype=torch.uint8, device=dev), torch.empty(scb, dtype=torch.uint8, device=dev),
            torch.zeros(2, dtype=torch.int64, device=dev))


B = {"local": bufs(d0), "peer": bufs(d1)}
B2 = {"local": bufs(d0), "peer": bufs(d1)}
out = torch.empty(n, dtype=torch.float32, device=d0)


def comp(where, src=x, b=B):
    blob, sc, ln = b[where]
    L.check(lib.gz_compress(src.data_ptr(), n, eb, 32, blob.data_ptr(), cap, ln.data_ptr(), sc.data_ptr(), None,
                            tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "c")


def dec(where):
    blob, sc, _ = B[where]
    L.check(lib.gz_decompress_sidecar(blob.data_ptr(), sc.data_ptr(), n, eb, out.data_ptr(), ws.status_ptr(), s), "d")


def step(src, dst):
    blob, sc, _ = B[src]
    ob, osc, oln = B2[dst]
    L.check(lib.gz_reduce_step(blob.data_ptr(), sc.data_ptr(), y.data_ptr(), n, eb, 0, None, ob.data_ptr(), cap,
                               oln.data_ptr(), osc.data_ptr(), tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "r")


def timeit(fn, reps=15):
    ts = []
    for it in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize(d0)
        if it >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


class _CI(__import__("ctypes").Structure):
    _fields_ = [("src", __import__("ctypes").c_void_p), ("dst", __import__("ctypes").c_void_p),
                ("d_len", __import__("ctypes").c_void_p), ("max_bytes", __import__("ctypes").c_uint64)]


def copy(src_where, dst_where):
    sb, _, sl = B[src_where]
    db, _, _ = B2[dst_where]
    it = (_CI * 1)(_CI(sb.data_ptr(), db.data_ptr(), sl.data_ptr(), cap))
    L.check(lib.gz_copy_items(it, 1, s), "copy")


def ce_copy(src_where, dst_where, nbytes):
    B2[dst_where][0][:nbytes].copy_(B[src_where][0][:nbytes], non_blocking=True)


comp("local"), comp("peer")
torch.cuda.synchronize(d0)
torch.cuda.synchronize(d1)
L_ = int(B["local"][2][0].item())
print(f"n=2^{n.bit_length() - 1} blob {L_} B CR {4 * n / L_:.3f}")
for name, fn in (("compress -> local", lambda: comp("local")), ("compress -> peer", lambda: comp("peer")),
                 ("decode local", lambda: dec("local")), ("decode peer blob", lambda: dec("peer")),
                 ("step local->local", lambda: step("local", "local")), ("step local->peer", lambda: step("local", "peer")),
                 ("step peer->local", lambda: step("peer", "local")),
                 ("copy kernel peer->local", lambda: copy("peer", "local")),
                 ("copy kernel local->peer", lambda: copy("local", "peer")),
                 ("CE copy peer->local", lambda: ce_copy("peer", "local", L_))):
    print(f"{name:22s} {timeit(fn):8.1f} us")
assert bytes(B["local"][0][:L_].cpu().numpy()) == bytes(B["peer"][0][:L_].cpu().numpy())
assert bytes(B2["local"][0][:64].cpu().numpy()) == bytes(B2["peer"][0][:64].cpu().numpy())
