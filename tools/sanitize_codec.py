"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): compress, decompress with sidecar, gz_index
on host bytes (+ truncated / corrupt blobs), fused reduce step (blob and
slotted I/O), decode+reduce, multi-segment compression, multi-blob decode,
fixed-rate codec, checked copy and apply_op.  Checks results against the
oracle so a silent corruption also fails."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from paper_2308_05199_b200 import collectives as C
from paper_2308_05199_b200.comm import _StepIO
from oracle import oracle as O

lib = L.lib()
ws = gz.Workspace()
n = 70_001
x = O.smooth_field(n) + np.random.default_rng(1).normal(0, 1e-3, n).astype(np.float32)
x[100:132] = np.float32(1e30)  # a raw block
ref = O.compress(x, 1e-4)
blob = gz.compress(torch.from_numpy(x).cuda(), 1e-4, ws, return_offsets=True)
assert bytes(blob) == ref
assert gz.decompress(blob, ws).cpu().numpy().tobytes() == O.decompress(ref).tobytes()
assert gz.decompress(ref, ws).tobytes() == O.decompress(ref).tobytes()  # gz_index path
for bad in (ref[:-7], ref[: 24 + 2048 * 5], ref + b"\x00"):
    try:
        gz.decompress(bad, ws)
    except gz.DecodeError:
        pass
y = O.smooth_field(n, 0.37)
outs = C.ring_allreduce_virtual([x, y, O.smooth_field(n, 0.9)], 1e-4, ws=ws)
exp = O.ring_allreduce([x, y, O.smooth_field(n, 0.9)], 1e-4)
assert all(a.cpu().numpy().tobytes() == b.tobytes() for a, b in zip(outs, exp))
rd = C.rd_allreduce_virtual([x, y, O.smooth_field(n, 0.9)], 1e-4, ws=ws)
assert all(a.cpu().numpy().tobytes() == b.tobytes() for a, b in zip(rd, O.rd_allreduce([x, y, O.smooth_field(n, 0.9)], 1e-4)))
sc = C.binomial_scatter_virtual(x, 5, 1e-4, root=2, ws=ws)
assert all(a.cpu().numpy().tobytes() == b.tobytes() for a, b in zip(sc, O.binomial_scatter(x, 5, 1e-4, root=2)))
# slotted step + step_reduce (the ring's intermediate messages)
xt = torch.from_numpy(x).cuda()
nt = int(lib.gz_num_tiles(n))
slots = torch.empty(int(lib.gz_slots_bytes(n)) + 128, dtype=torch.uint8, device="cuda")
base = (slots.data_ptr() + 127) & ~127
sizes = torch.empty(nt, dtype=torch.int32, device="cuda")
widths = torch.empty(32 * nt, dtype=torch.uint8, device="cuda")
io = _StepIO()
io.out_slots, io.out_sizes, io.out_widths = base, sizes.data_ptr(), widths.data_ptr()
tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
s = torch.cuda.current_stream().cuda_stream
L.check(lib.gz_step(ctypes.byref(io), xt.data_ptr(), n, 1e-4, 0, None, tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_step")
io2 = _StepIO()
io2.in_slots, io2.in_sizes, io2.in_widths = base, sizes.data_ptr(), widths.data_ptr()
ys = torch.empty(n, dtype=torch.float32, device="cuda")
L.check(lib.gz_step_reduce(ctypes.byref(io2), None, n, 1e-4, 0, ys.data_ptr(), ws.status_ptr(), s), "gz_step_reduce")
torch.cuda.synchronize()
assert ys.cpu().numpy().tobytes() == O.decompress(ref).tobytes()
for b in (4, 11):
    fr = gz.fixed_rate_compress(x[:5000] if b == 4 else np.zeros(33, np.float32), b, ws)
    assert fr == O.fixed_rate_compress(x[:5000] if b == 4 else np.zeros(33, np.float32), b)
z = C.apply_op("max", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
assert z.cpu().numpy().tobytes() == np.where(np.isnan(x) | (x > y), x, y).astype(np.float32).tobytes()
torch.cuda.synchronize()
print("sanitize run ok")
