"""A/B of libgzccl.so builds on the cfg1 field (2^24, L2 flushed) and 2^27: compress /
decompress medians (CUDA events; the builds are interleaved every iteration so clock
drift hits all alike), 10 back-to-back compresses, the live per-kernel durations
(torch.profiler / CUPTI) and byte equality of every build's blob and decode with the
FIRST build's (the shipped, oracle-checked one).
python tools/exp/ab_codec2.py base.so new.so [...]   (EBS=1e-4,1e-3 NS=24,27)"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from oracle import oracle as O

u64, u32, p, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double
libs = {}
for path in sys.argv[1:]:
    L = ctypes.CDLL(path)
    L.gz_compress.argtypes = [p, u64, dbl, u32, p, u64, p, p, p, p, u64, p, p]
    L.gz_compress_bound.restype = L.gz_workspace_bytes.restype = L.gz_sidecar_bytes.restype = u64
    L.gz_compress_bound.argtypes = L.gz_workspace_bytes.argtypes = L.gz_sidecar_bytes.argtypes = [u64]
    L.gz_workspace_init.argtypes = [p, u64, p]
    L.gz_decompress_sidecar.argtypes = [p, p, u64, dbl, p, p, p]
    libs[os.path.basename(path)] = L
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
EBS = [float(e) for e in os.environ.get("EBS", "1e-4").split(",")]
NS = [1 << int(k) for k in os.environ.get("NS", "24,27").split(",")]
ITERS = int(os.environ.get("ITERS", "15"))


def ev_time(fn, do_flush=True):
    if do_flush:
        flush.zero_(); flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    rc = fn()
    b.record(s)
    torch.cuda.synchronize()
    assert rc == 0, rc
    return a.elapsed_time(b) * 1e3


for n in NS:
  x = torch.from_numpy(O.smooth_field(n)).cuda()
  for eb in EBS:
    st_ = {}
    for name, L in libs.items():
        d = {}
        cap = L.gz_compress_bound(n)
        d["blob"] = blob = torch.empty(cap, dtype=torch.uint8, device="cuda")
        d["sc"] = sc = torch.empty(L.gz_sidecar_bytes(n), dtype=torch.uint8, device="cuda")
        wsb = L.gz_workspace_bytes(n)
        d["ws"] = ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        L.gz_workspace_init(ws.data_ptr(), wsb, s.cuda_stream)
        d["st"] = st = torch.full((8,), -1, dtype=torch.int64, device="cuda")
        d["y"] = y = torch.empty(n, dtype=torch.float32, device="cuda")
        d["comp"] = (lambda L=L, blob=blob, cap=cap, st=st, sc=sc, ws=ws, wsb=wsb:
                     L.gz_compress(x.data_ptr(), n, eb, 32, blob.data_ptr(), cap, st.data_ptr() + 32, sc.data_ptr(),
                                   None, ws.data_ptr(), wsb, st.data_ptr(), s.cuda_stream))
        d["dec"] = (lambda L=L, blob=blob, sc=sc, y=y, st=st:
                    L.gz_decompress_sidecar(blob.data_ptr(), sc.data_ptr(), n, eb, y.data_ptr(), st.data_ptr(), s.cuda_stream))
        d["tc"], d["td"] = [], []
        st_[name] = d
    names = list(libs)
    for it in range(ITERS):
        order = names[it % len(names):] + names[:it % len(names)]
        for nm in order:
            d = st_[nm]
            tc = ev_time(d["comp"]); td = ev_time(d["dec"])
            if it >= 3:
                d["tc"].append(tc); d["td"].append(td)
    ref = None
    for nm in names:
        d = st_[nm]
        # 10 back-to-back compresses (no flush in between)
        bb = ev_time(lambda: sum(d["comp"]() for _ in range(10))) / 10
        ln = int(d["st"][4].item())
        hb, hy = d["blob"][:ln].cpu(), d["y"].cpu()
        if ref is None:
            ref, same = (hb, hy), "base"
        else:
            same = "EQUAL" if (hb.numel() == ref[0].numel() and torch.equal(hb, ref[0]) and torch.equal(hy.view(torch.int32), ref[1].view(torch.int32))) else "DIFFERENT"
        kern = ""
        try:
            from torch.profiler import profile, ProfilerActivity
            flush.zero_(); flush.sum(); torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                d["comp"](); d["dec"]()
                torch.cuda.synchronize()
            evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "gz" in e.name]
            kern = "  ".join("%s %.1f" % (e.name.split("<")[0].split("(")[0].replace("void ", "").replace("gz::", ""),
                                          e.time_range.elapsed_us()) for e in evs)
        except Exception as ex:
            kern = "profiler: %s" % ex
        c, dd = sorted(d["tc"]), sorted(d["td"])
        print(f"n=2^{n.bit_length()-1} eb={eb:g} {nm:16s} compress med {c[len(c)//2]:7.1f} min {c[0]:7.1f} b2b {bb:6.1f} | "
              f"decompress med {dd[len(dd)//2]:7.1f} min {dd[0]:7.1f} | len {ln} {same} | {kern}", flush=True)
