"""Allgather decode reading an owner's slotted message out of a PEER GPU's
memory (single process, two GPUs, peer access), as Communicator's "slots"
allgather does, in a form ncu can replay: GPU 0 compresses chunk A into
slotted form; GPU 1 decodes it with gz_decompress_slots_multi over NVLink.
Also times the same decode from GPU 1's own copy of the slots (local HBM).
python tools/prof_peer_decode.py [n] [reps]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_05199_b200 as gz
from paper_2308_05199_b200 import _lib as L
from paper_2308_05199_b200.comm import _StepIO
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = L.lib()
nt = int(lib.gz_num_tiles(n))


def slots_on(dev):
    sl = torch.empty(int(lib.gz_slots_bytes(n)) + 128, dtype=torch.uint8, device=dev)
    return sl, torch.empty(nt, dtype=torch.int32, device=dev), torch.empty(32 * nt, dtype=torch.uint8, device=dev)


al = lambda t: (t.data_ptr() + 127) & ~127  # noqa: E731
torch.cuda.set_device(0)
ws0 = gz.Workspace("cuda:0")
a = torch.from_numpy(O.smooth_field(n)).to("cuda:0")
s0 = slots_on("cuda:0")
io = _StepIO()
io.out_slots, io.out_sizes, io.out_widths = al(s0[0]), s0[1].data_ptr(), s0[2].data_ptr()
tws0 = ws0.tile_ws(int(lib.gz_workspace_bytes(n)))
L.check(lib.gz_step(ctypes.byref(io), a.data_ptr(), n, 1e-4, 0, None, tws0.data_ptr(), tws0.numel(), ws0.status_ptr(),
                    torch.cuda.current_stream(0).cuda_stream), "gz_step")
torch.cuda.synchronize(0)
torch.cuda.set_device(1)
L.check(lib.gz_enable_peer_access(0), "gz_enable_peer_access")
ws1 = gz.Workspace("cuda:1")
b = torch.from_numpy(O.smooth_field(n, 0.37)).to("cuda:1")
s1 = slots_on("cuda:1")
tws1 = ws1.tile_ws(int(lib.gz_workspace_bytes(n)))
st = torch.cuda.current_stream(1)
y = torch.empty(n, dtype=torch.float32, device="cuda:1")
local = tuple(t.to("cuda:1") for t in s0)  # the same slots in GPU 1's memory


def decode(slots):
    P = ctypes.c_void_p * 1
    L.check(lib.gz_decompress_slots_multi(P(al(slots[0])), P(slots[1].data_ptr()), P(slots[2].data_ptr()),
                                          (ctypes.c_uint64 * 1)(n), 1, 1e-4, P(y.data_ptr()), 0, ws1.status_ptr(),
                                          st.cuda_stream), "gz_decompress_slots_multi")


outs = {}
for name, sl in (("peer", s0), ("local", local)):
    ts = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        decode(sl)
        e1.record(st)
        torch.cuda.synchronize(1)
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name} slots decode n={n}: {sorted(ts)[len(ts) // 2]:.1f} us (median of {reps})", flush=True)
    outs[name] = y.clone()
assert torch.equal(outs["peer"], outs["local"]), "peer and local decodes differ"
