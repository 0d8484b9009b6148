"""NVLink pull bandwidth: copy kernel (various SM budgets) and copy engine, from 1 and
from 3 peers at once.  One process, GPUs 0..3.  python tools/exp/peer_copy.py [MB]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2308_05199_b200 import _lib as L

lib = L.lib()
MB = int(sys.argv[1]) if len(sys.argv) > 1 else 21
nb = MB << 20
ng = torch.cuda.device_count()
torch.cuda.set_device(0)
for p in range(1, ng):
    L.check(lib.gz_enable_peer_access(p), "peer")
src = [torch.ones(nb, dtype=torch.uint8, device=f"cuda:{p}") for p in range(ng)]
dst = [torch.empty(nb, dtype=torch.uint8, device="cuda:0") for _ in range(ng)]
streams = [torch.cuda.Stream(device=0) for _ in range(ng)]


class CI(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("d_len", ctypes.c_void_p), ("max_bytes", ctypes.c_uint64)]


def kcopy(p, budget, st):
    it = (CI * 1)(CI(src[p].data_ptr(), dst[p].data_ptr(), None, nb))
    L.check(lib.gz_copy_items_sms(it, 1, budget, st.cuda_stream), "copy")


def timeit(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        torch.cuda.synchronize(0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize(0)
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


cur = torch.cuda.current_stream(0)


def par(fns):
    ev = torch.cuda.Event()
    ev.record(cur)
    for k, f in enumerate(fns):
        streams[k].wait_stream(cur)
        f(streams[k])
    for k in range(len(fns)):
        cur.wait_stream(streams[k])


for budget in (0, 24, 48, 96):
    t = timeit(lambda: kcopy(1, budget, cur))
    print(f"kernel copy 1 peer, {MB} MB, sms budget {budget}: {t:.1f} us = {nb / t / 1e3:.0f} GB/s", flush=True)
t = timeit(lambda: dst[1].copy_(src[1], non_blocking=True))
print(f"CE copy 1 peer: {t:.1f} us = {nb / t / 1e3:.0f} GB/s")
if ng >= 4:
    for budget in (16, 24, 48):
        t = timeit(lambda: par([lambda st, p=p: kcopy(p, budget, st) for p in (1, 2, 3)]))
        print(f"kernel copy 3 peers concurrently, budget {budget} each: {t:.1f} us = {3 * nb / t / 1e3:.0f} GB/s")

    def ce3(st_list=None):
        def f(st, p):
            with torch.cuda.stream(st):
                dst[p].copy_(src[p], non_blocking=True)
        par([lambda st, p=p: f(st, p) for p in (1, 2, 3)])
    t = timeit(ce3)
    print(f"CE copy 3 peers concurrently: {t:.1f} us = {3 * nb / t / 1e3:.0f} GB/s")
