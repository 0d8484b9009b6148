"""Benchmark driver (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--sweep]

BASELINE.json metric: "gZ-Allreduce effective GB/s at 1-8 B200 vs NCCL;
compressor HBM GB/s".

* N = 1  -> configs[0]: compress/decompress round trip of the synthetic smooth
  float32 field (2^24 values, eb = 1e-4, block 32).  ``value`` = codec HBM
  GB/s of the round trip = algorithmic bytes (4n + |blob| per compress,
  |blob| + 4n per decompress) / device time (CUDA events); the compressor
  alone is ``detail.compressor_hbm_gbs`` and the line's ``roofline``.  L2
  (126 MB) is flushed before every timed step.
* N > 1  -> configs[1]: compressed ring Allreduce (compressed reduce-scatter +
  compress-once allgather) of a 512 MiB float32 field per rank, eb = 1e-4,
  one process per GPU over NVLink peer memory; ``value`` = effective GB/s =
  uncompressed bytes per rank / max-over-ranks device time (NCCL's algbw).
  NCCL all_reduce, the cfg3 1 GiB binomial scatter (vs NCCL scatter) and
  recursive doubling are measured alongside (``detail``).
* ``--sweep`` (N > 1) -> configs[3]: the allreduce message-size sweep, 1 MiB ..
  2 GiB per rank x eb in {1e-2, 1e-3, 1e-4}, one JSON line per point, NCCL
  all_reduce at each size.

Every timed output is checked against the CPU oracle (C restatement of the
reference codec / schedules, all host threads) OUTSIDE the timed region;
the line's ``parity`` key says what was compared.

``--impl reference`` times the reference algorithm on the host CPU (the C
restatement in oracle/, all host threads; the reference's own numpy code is
the same algorithm single-threaded) on the same metric, config and unit.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gZ-Allreduce effective GB/s at 1-8 B200 vs NCCL; compressor HBM GB/s"
EB = 1e-4
N_CFG1 = 1 << 24
S_CFG2 = 512 << 20  # bytes per rank
N_CFG3 = 1 << 28    # values at the scatter root (1 GiB)
DTYPE = "f32 values, u8 compressed wire, f64 closed-loop quantiser"


def shared_config(n_gpus: int, per_rank_bytes: int = S_CFG2) -> dict:
    """The workload, identical in both arms' lines (numbers that only one arm
    measures go under ``detail``)."""
    if n_gpus <= 1:
        return {"workload": "cfg1 compress/decompress round trip, 2^24 f32, eb=1e-4, block=32",
                "values": N_CFG1, "eb": EB, "block": 32,
                "l2": "flushed before every timed step (256 MB write + 256 MB read)"}
    return {"workload": f"ring-allreduce (compressed RS + compress-once AG), {per_rank_bytes >> 20} MiB f32 per rank, "
                        "eb=1e-4", "bytes_per_rank": per_rank_bytes, "eb": EB, "ranks": n_gpus,
            "parallelism": f"ring over {n_gpus} ranks", "l2": "inputs (512 MiB per rank) larger than L2"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                self.samples.append([v.strip() for v in out.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        import statistics

        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _line(n_gpus, steps, warmup, value, ms, config, **extra) -> dict:
    d = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n_gpus, "steps": steps, "warmup": warmup,
         "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
         "data": "synthetic smooth field 0.5 sin(2 pi i/65536 + p) + 0.25 sin(2 pi i/4099 + p), p = 0.37 rank",
         "config": config}
    d.update(extra)
    return d


# ---------------------------------------------------------------------------
# CPU reference arm (C restatement of the reference algorithm, all host threads)
# ---------------------------------------------------------------------------


def cpu_codec_round_trip(x, eb: float, threads: int):
    from oracle import oracle as O

    t0 = time.perf_counter()
    blob = O.compress(x, eb, threads=threads)
    O.decompress(blob, threads=threads)
    dt = time.perf_counter() - t0
    return 2 * (4 * x.size + len(blob)) / dt / 1e9, dt


def cfg2_inputs(N: int, n: int):
    from oracle import oracle as O

    return [O.smooth_field(n, 0.37 * r) for r in range(N)]


def cpu_ring_allreduce(bufs, threads: int):
    """One host ring allreduce of the per-rank buffers (the reference schedule,
    collectives.py:294-308, every codec call on all threads): (outputs, secs)."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    outs = O.ring_allreduce(bufs, EB, threads=threads)
    return outs, time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU, same metric and config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O

    threads = cpu_threads()
    N = max(1, args.gpus)
    if N == 1:
        x = O.smooth_field(N_CFG1)
        for _ in range(max(1, min(args.warmup, 2))):
            cpu_codec_round_trip(x, EB, threads)
        ts = [cpu_codec_round_trip(x, EB, threads)[1] for _ in range(args.steps)]
        t = sum(ts) / len(ts)
        blob_len = len(O.compress(x, EB, threads=threads))
        gbs = 2 * (4 * N_CFG1 + blob_len) / t / 1e9
        sample = "full cfg1 field (2^24 f32) every step"
    else:
        # full cfg2 (512 MiB per rank) unless K steps of it would exceed ~4 minutes;
        # then each step is a bounded sample (smaller per-rank buffer, same schedule)
        n = S_CFG2 // 4
        bufs = cfg2_inputs(N, n)
        _, t1 = cpu_ring_allreduce(bufs, threads)  # warm-up step, also the time estimate
        while n > (1 << 20) and t1 * (args.steps + 1) > 240.0:
            n //= 2
            t1 /= 2
        bufs = [b[:n] for b in bufs]
        ts = [cpu_ring_allreduce(bufs, threads)[1] for _ in range(args.steps)]
        t = sum(ts) / len(ts)
        gbs = 4 * n / t / 1e9
        sample = (f"{4 * n >> 20} MiB per rank, {N} ranks simulated on the host"
                  + ("" if n == S_CFG2 // 4 else " (bounded sample of the 512 MiB workload)"))
    base = {"value": round(gbs, 5), "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample,
            "cpu": cpu_model()}
    line = _line(N, args.steps, args.warmup, round(gbs, 5), round(t * 1e3, 3), shared_config(N), impl="reference",
                 cpu_baseline=base,
                 e2e={"value": round(gbs, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm, N = 1: codec round trip
# ---------------------------------------------------------------------------


def _traffic(key: str):
    """DRAM bytes per launch of the line's dominant kernel, from the committed ncu capture
    (profiles/traffic.json, with the command and capture it came from); None if absent."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(tp) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def _issue_roofline(t_compress: float):
    """The compressor's instruction-issue floor: warp-instructions per call
    from the committed ncu capture / (SMs x 4 schedulers x SM clock), against the measured
    compress time."""
    ins = _traffic("compress_cfg1_warp_instructions")
    if not ins:
        return None
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk_hz = 1.965e9  # B200 boost clock (the bench's clock sampler shows 1965 MHz under load)
    floor = ins / (sms * 4 * clk_hz)
    return {"warp_instructions_per_call": ins, "issue_floor_us": round(floor * 1e6, 2),
            "frac": round(floor / t_compress, 4), "source": "profiles/traffic.json (ncu instruction counts)"}


def e2e_codec(gz, xp, ws_list, streams, total_steps: int, ref_blob: bytes):
    """End to end through the public API from pinned host memory: each step =
    compress(pinned f32 host tensor) -> pinned host blob (H2D of the input, the
    kernels, D2H of the blob), then decompress(host blob) -> pinned host f32
    (H2D of the blob, device indexing of the reference bytes, decode, D2H).
    Several steps are in flight on as many streams (separate workspaces), so one
    step's H2D overlaps another's D2H on the full-duplex link."""
    import torch

    lanes = len(streams)
    res = [None] * lanes
    barrier = threading.Barrier(lanes + 1)

    def worker(k):
        barrier.wait()
        b = y = None
        for _ in range(k, total_steps, lanes):
            b = gz.compress(xp, EB, ws_list[k], stream=streams[k])
            y = gz.decompress(b, ws_list[k], stream=streams[k])
        res[k] = (b, y)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(lanes)]
    for t in th:
        t.start()
    torch.cuda.synchronize()
    barrier.wait()
    t0 = time.perf_counter()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    for b, y in res:
        if b is not None:
            assert b.numpy().tobytes() == ref_blob, "e2e blob differs from the oracle"
    return wall, res[0][1]


def bench_codec(args):
    import numpy as np
    import torch

    import paper_2308_05199_b200 as gz
    from paper_2308_05199_b200 import _lib as L
    from oracle import oracle as O

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    lib = L.lib()
    n = N_CFG1
    xh = O.smooth_field(n)
    x = torch.from_numpy(xh).to(dev)
    ws = gz.Workspace(dev)
    blob0 = gz.compress(x, EB, ws)
    Lb = len(blob0)
    # persistent buffers for the timed loop (the public API allocates per call)
    cap = int(lib.gz_compress_bound(n))
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    sc = torch.empty(int(lib.gz_sidecar_bytes(n)), dtype=torch.uint8, device=dev)
    tws = ws.tile_ws(int(lib.gz_workspace_bytes(n)))
    y = torch.empty(n, dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(256 << 20, dtype=torch.uint8, device=dev).view(torch.int64)
    stream = torch.cuda.current_stream()

    def l2_flush():
        # 256 MB write (> 126 MB L2), then a 256 MB read: the read evicts the
        # write's dirty lines, so their write-back does not land inside the
        # timed region and L2 holds none of the step's data
        flush.zero_()
        flush_r.sum()
    s = stream.cuda_stream

    def comp():
        L.check(lib.gz_compress(x.data_ptr(), n, EB, 32, out.data_ptr(), cap, ws.len_ptr(), sc.data_ptr(), None,
                                tws.data_ptr(), tws.numel(), ws.status_ptr(), s), "gz_compress")

    def dec():
        L.check(lib.gz_decompress_sidecar(out.data_ptr(), sc.data_ptr(), n, EB, y.data_ptr(), ws.status_ptr(), s),
                "gz_decompress_sidecar")

    warm = max(args.warmup, 3)
    for _ in range(warm):
        l2_flush()
        comp()
        dec()
    torch.cuda.synchronize()
    tc, td = [], []
    launches0 = int(lib.gz_launch_count())
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            l2_flush()  # outside the timed events
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            comp()
            e1.record(stream)
            dec()
            e2.record(stream)
            torch.cuda.synchronize()
            tc.append(e0.elapsed_time(e1) * 1e-3)
            td.append(e1.elapsed_time(e2) * 1e-3)
    torch.cuda.synchronize()
    launches = int(lib.gz_launch_count()) - launches0
    # parity (outside the timed region): the blob of the LAST timed call and its decoded
    # values are byte-compared with the CPU oracle (C restatement of codec.py, all host threads)
    thr_all = cpu_threads()
    ref_blob = O.compress(xh, EB, threads=thr_all)
    assert int(ws.status[4].item()) == len(ref_blob), "timed blob length differs from the oracle"
    assert out[:Lb].cpu().numpy().tobytes() == ref_blob, "timed blob differs from the oracle"
    ref_y = O.decompress(ref_blob, threads=thr_all)
    assert y.cpu().numpy().tobytes() == ref_y.tobytes(), "decode differs"
    parity = {"cfg1": "bit-exact vs oracle (blob + decoded values of the last timed step)"}
    t_c, t_d = sum(tc) / len(tc), sum(td) / len(td)
    bytes_c = 4 * n + Lb
    bytes_d = Lb + 4 * n
    value = (bytes_c + bytes_d) / (t_c + t_d) / 1e9
    peak, peak_kind = peaks()
    achieved_c = bytes_c / t_c / 1e9

    # supplementary: the codec on a field larger than L2 (2^27 values, 512 MB;
    # same synthetic field, no flush needed), where the per-call fixed cost no
    # longer dominates -- reported under detail, not as the line's value
    big = {}
    try:
        nb = 1 << 27
        xbh = O.smooth_field(nb)
        xb = torch.from_numpy(xbh).to(dev)
        capb = int(lib.gz_compress_bound(nb))
        outb = torch.empty(capb, dtype=torch.uint8, device=dev)
        scb = torch.empty(int(lib.gz_sidecar_bytes(nb)), dtype=torch.uint8, device=dev)
        twb = gz.Workspace(dev)
        twb.reset_status()
        twsb = twb.tile_ws(int(lib.gz_workspace_bytes(nb)))
        yb_ = torch.empty(nb, dtype=torch.float32, device=dev)

        def comp_b():
            L.check(lib.gz_compress(xb.data_ptr(), nb, EB, 32, outb.data_ptr(), capb, twb.len_ptr(), scb.data_ptr(),
                                    None, twsb.data_ptr(), twsb.numel(), twb.status_ptr(), s), "gz_compress")

        def dec_b():
            L.check(lib.gz_decompress_sidecar(outb.data_ptr(), scb.data_ptr(), nb, EB, yb_.data_ptr(),
                                              twb.status_ptr(), s), "gz_decompress_sidecar")
        for _ in range(3):
            comp_b()
            dec_b()
        torch.cuda.synchronize()
        Lbb = int(twb.status[4].item())
        tcb, tdb = [], []
        for _ in range(max(5, min(args.steps, 20))):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            comp_b()
            e1.record(stream)
            dec_b()
            e2.record(stream)
            torch.cuda.synchronize()
            tcb.append(e0.elapsed_time(e1) * 1e-3)
            tdb.append(e1.elapsed_time(e2) * 1e-3)
        tcb_m, tdb_m = sorted(tcb)[len(tcb) // 2], sorted(tdb)[len(tdb) // 2]
        refb = O.compress(xbh, EB, threads=thr_all)
        assert Lbb == len(refb) and outb[:Lbb].cpu().numpy().tobytes() == refb, "2^27 blob differs from the oracle"
        assert yb_.cpu().numpy().tobytes() == O.decompress(refb, threads=thr_all).tobytes(), "2^27 decode differs"
        parity["codec_2p27"] = "bit-exact vs oracle"
        big = {"values": nb, "compressed_bytes": Lbb, "compress_us": round(tcb_m * 1e6, 1),
               "decompress_us": round(tdb_m * 1e6, 1),
               "compress_hbm_gbs": round((4 * nb + Lbb) / tcb_m / 1e9, 1),
               "compress_frac": round((4 * nb + Lbb) / tcb_m / 1e9 / peak, 4),
               "decompress_hbm_gbs": round((4 * nb + Lbb) / tdb_m / 1e9, 1),
               "decompress_frac": round((4 * nb + Lbb) / tdb_m / 1e9 / peak, 4), "stat": "median"}
        del xb, outb, scb, twsb, yb_, refb
    except AssertionError:
        raise
    except Exception as e:  # a supplementary number must not sink the line
        big = {"error": str(e)[:200]}
    torch.cuda.empty_cache()

    # e2e through the public API with pinned host buffers, several steps in flight
    xp = torch.from_numpy(xh).pin_memory()
    # steps in flight: tools/exp/e2e_var.py, six runs each after warm-up: 2 lanes 63-66 GB/s,
    # 3 lanes 72-81, 4 lanes 76-83 (the first run after a short warm-up collapses while the
    # pinned host pools fill, hence the longer warm-up)
    lanes = 4
    e2e_ws = [gz.Workspace(dev) for _ in range(lanes)]
    e2e_streams = [torch.cuda.Stream(dev) for _ in range(lanes)]
    e2e_steps = max(8, min(2 * args.steps, 40))
    for _ in range(2):  # warm-up (pinned host pools, index workspaces)
        e2e_codec(gz, xp, e2e_ws, e2e_streams, 3 * lanes, ref_blob)
    # three timed runs of e2e_steps steps each; the median run is reported (the host side
    # of the copies varies from run to run, tools/exp/e2e_var.py)
    runs = []
    for _ in range(3):
        wall_r, y_last = e2e_codec(gz, xp, e2e_ws, e2e_streams, e2e_steps, ref_blob)
        assert y_last.numpy().tobytes() == ref_y.tobytes(), "e2e decode differs from the oracle"
        runs.append(wall_r)
    wall = sorted(runs)[1]
    parity["e2e"] = "bit-exact vs oracle (host blob and host values)"
    e2e = e2e_steps * (bytes_c + bytes_d) / wall / 1e9

    # CPU baseline (oracle port, all host threads) on the same workload
    cpu_gbs, cpu_t = cpu_codec_round_trip(xh, EB, thr_all)
    cpu_gbs2, cpu_t2 = cpu_codec_round_trip(xh, EB, thr_all)
    cpu_gbs = max(cpu_gbs, cpu_gbs2)

    traffic = _traffic("compress_cfg1")
    line = _line(
        1, args.steps, warm, round(value, 2), round((t_c + t_d) * 1e3, 5), shared_config(1),
        detail={"value_is": "codec round trip: (bytes of compress + bytes of decompress) / (compress + decompress "
                            "device time)", "compressed_bytes": Lb, "compression_ratio": round(4 * n / Lb, 4),
                "compress_us": round(t_c * 1e6, 2), "decompress_us": round(t_d * 1e6, 2),
                "compressor_hbm_gbs": round(achieved_c, 1), "decompressor_hbm_gbs": round(bytes_d / t_d / 1e9, 1),
                "codec_2p27": big,
                "issue_roofline": _issue_roofline(t_c)},
        roofline={"bound": "hbm", "kernel": "compressor (k_tile_encode + k_gather)", "achieved": round(achieved_c, 1),
                  "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved_c / peak, 4),
                  "traffic": traffic, "algorithmic_bytes_per_launch": bytes_c,
                  "bytes_per_unit": "4 B per input value + compressed bytes (SURVEY 8(d))"},
        cpu_baseline={"value": round(cpu_gbs, 4), "unit": "GB/s", "cores": thr_all, "kind": "port",
                      "sample": f"full cfg1 field, best of 2 round trips, C oracle with {thr_all} threads",
                      "cpu": cpu_model()},
        e2e={"value": round(e2e, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n + Lb, "d2h_bytes_per_step": Lb + 4 * n,
             "api": "compress(pinned host f32 tensor) -> pinned host blob; decompress(host blob) -> pinned host f32; "
                    f"{lanes} steps in flight on {lanes} streams", "wall_ms_per_step": round(wall / e2e_steps * 1e3, 3),
             "steps": e2e_steps, "runs": 3, "stat": "median run",
             "run_gbs": [round(e2e_steps * (bytes_c + bytes_d) / w / 1e9, 2) for w in runs]},
        gpu_launches=launches, clocks=clk.summary(), parity=parity)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm, N > 1: compressed ring allreduce over NVLink peer memory
# ---------------------------------------------------------------------------


def _max_over_ranks(v: float, dev) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], device="cpu" if dist.get_backend() == "gloo" else dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _digest(t) -> str:
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()


def _init_dist():
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # more ranks than GPUs (tools/gpu_n8_rehearsal.sh): ranks share GPUs, NCCL (one rank
    # per GPU) is replaced by gloo for the object plumbing and the NCCL comparators are
    # skipped; the numbers of such a run are a code-path rehearsal, not a measurement
    oversub = world > torch.cuda.device_count()
    local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    return rank, world, local, dev, oversub


def _timed_calls(fn, stream, reps, dev):
    """Median device time of `reps` calls (barrier + sync around each), max over ranks."""
    import torch
    import torch.distributed as dist

    ts = []
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return _max_over_ranks(ts[len(ts) // 2], dev)


def bench_allreduce(args):
    import torch
    import torch.distributed as dist

    from paper_2308_05199_b200 import _lib as L
    from paper_2308_05199_b200 import comm
    from paper_2308_05199_b200.collectives import chunk_spans
    from oracle import oracle as O

    rank, world, local, dev, oversub = _init_dist()
    lib = L.lib()
    n = S_CFG2 // 4
    xh = O.smooth_field(n, 0.37 * rank)
    x = torch.from_numpy(xh).to(dev)
    c = comm.Communicator(dist.group.WORLD, dev)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def ev():
        return torch.cuda.Event(enable_timing=True)

    warm = max(args.warmup, 3)
    for _ in range(warm):
        c.ring_allreduce(x, EB, out=out, check=False)
    c.check()
    dist.barrier()
    times, step_t = [], []
    launches0 = int(lib.gz_launch_count()) + c.graph_launches
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record(stream)
            c.ring_allreduce(x, EB, out=out, check=False)  # errors are checked once after the loop
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
    launches = int(lib.gz_launch_count()) + c.graph_launches - launches0  # eager launches + graph replays
    c.check()  # every rank: no non-finite input, decode or peer-flag error in the timed calls
    out_digest = _digest(out)
    # fused-step kernel durations: CUDA-event marks after every wait/launch of
    # the same call, on extra calls after the timed loop (marks perturb timing)
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        c.events = []
        c.ring_allreduce(x, EB, out=out, check=False)
        torch.cuda.synchronize()
        marks = c.events
        for (_, a), (lab, b) in zip(marks, marks[1:]):
            if lab in ("reduce", "reduce_last"):
                step_t.append(a.elapsed_time(b) * 1e-3)
        c.events = None
    t = _max_over_ranks(sum(times) / len(times), dev)
    cr = c.compression_ratio()
    m = n // world
    t_step = sum(step_t) / len(step_t)
    step_bytes = 4 * m + 2 * 4 * m / (cr or 1.0)  # local chunk + received blob + produced blob
    step_gbs = _max_over_ranks(-step_bytes / t_step / 1e9, dev) * -1.0  # slowest rank

    # e2e: pinned host input -> H2D -> allreduce -> D2H of the result, per step; consecutive
    # steps are pipelined on three streams with double-buffered device tensors (step i+1's H2D
    # and step i-1's D2H run beside step i's allreduce)
    xp = torch.from_numpy(xh).pin_memory()
    outp = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
    xd = [x, torch.empty_like(x)]
    od = [out, torch.empty_like(out)]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    in_ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    drained = [torch.cuda.Event() for _ in range(2)]

    def e2e_steps(k):
        for i in range(k):
            b = i & 1
            with torch.cuda.stream(h2d):
                h2d.wait_event(done[b])  # the previous allreduce on xd[b] has finished reading it
                xd[b].copy_(xp, non_blocking=True)
                in_ready[b].record(h2d)
            stream.wait_event(in_ready[b])
            stream.wait_event(drained[b])  # od[b] of step i-2 has been copied out
            c.ring_allreduce(xd[b], EB, out=od[b], check=False)
            done[b].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done[b])
                outp[b].copy_(od[b], non_blocking=True)
                drained[b].record(d2h)

    e2e_k = max(4, min(args.steps, 10))
    e2e_steps(4)  # warm-up: captures the graphs of both buffer pairs
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0 = ev()
    e0.record(stream)
    e2e_steps(e2e_k)
    stream.wait_stream(d2h)
    e1 = ev()
    e1.record(stream)
    torch.cuda.synchronize()
    c.check()
    t_e2e = _max_over_ranks(e0.elapsed_time(e1) * 1e-3 / e2e_k, dev)
    e2e_digest = hashlib.sha256(outp[(e2e_k - 1) & 1].numpy().tobytes()).hexdigest()

    # NCCL all_reduce comparator on the same tensor
    nccl_gbs = nccl_scatter_gbs = None
    if not oversub:
        y = x.clone()
        for _ in range(3):
            dist.all_reduce(y)
        tn = _timed_calls(lambda: dist.all_reduce(y), stream, max(3, min(args.steps, 10)), dev)
        nccl_gbs = round(S_CFG2 / tn / 1e9, 2)
        del y

    # configs[2]: binomial-tree compressed Scatter of a 1 GiB root buffer vs NCCL scatter
    ns = N_CFG3
    root_h = O.smooth_field(ns, 0.0) if rank == 0 else None
    root_buf = torch.from_numpy(root_h).to(dev) if rank == 0 else None
    lo_, hi_ = chunk_spans(ns, world)[rank]
    sc_out = torch.empty(hi_ - lo_, dtype=torch.float32, device=dev)
    for _ in range(3):
        c.binomial_scatter(root_buf, EB, root=0, out=sc_out, check=False)
    c.check()
    ts_ = _timed_calls(lambda: c.binomial_scatter(root_buf, EB, root=0, out=sc_out, check=False), stream,
                       max(3, min(args.steps, 10)), dev)
    c.check()
    scatter_gbs = 4 * ns / ts_ / 1e9
    sc_digest = _digest(sc_out)
    if not oversub:
        parts = list(root_buf[: (ns // world) * world].chunk(world)) if rank == 0 else None
        ys = torch.empty(ns // world, dtype=torch.float32, device=dev)
        for _ in range(3):
            dist.scatter(ys, parts, src=0)
        tns = _timed_calls(lambda: dist.scatter(ys, parts, src=0), stream, max(3, min(args.steps, 10)), dev)
        nccl_scatter_gbs = round(4 * ns / tns / 1e9, 2)
        del parts, ys
    del root_buf

    # recursive-doubling allreduce (the paper's gZ-Allreduce(ReDoub)) on the same tensors
    rdo = torch.empty_like(x)
    for _ in range(3):
        c.rd_allreduce(x, EB, out=rdo, check=False)
    trd = _timed_calls(lambda: c.rd_allreduce(x, EB, out=rdo, check=False), stream, max(3, min(args.steps, 10)), dev)
    c.check()
    rd_gbs = S_CFG2 / trd / 1e9
    del rdo
    torch.cuda.empty_cache()

    # parity + CPU baseline (outside every timed region): rank 0 runs the reference schedule
    # for all ranks on the host (C oracle, all threads) and compares every rank's output digest
    digests = [None] * world
    dist.all_gather_object(digests, (out_digest, e2e_digest, sc_digest))
    parity, cpu_base = None, None
    if rank == 0:
        thr = cpu_threads()
        outs, t_cpu = cpu_ring_allreduce(cfg2_inputs(world, n), thr)
        expect = [hashlib.sha256(o.tobytes()).hexdigest() for o in outs]
        del outs
        bad = [r for r in range(world) if digests[r][0] != expect[r] or digests[r][1] != expect[r]]
        sc_exp = O.binomial_scatter(root_h, world, EB, root=0, threads=thr)
        bad_sc = [r for r in range(world) if digests[r][2] != hashlib.sha256(sc_exp[r].tobytes()).hexdigest()]
        del sc_exp
        parity = {"ring_allreduce_512MiB": "bit-exact vs oracle on every rank (timed and e2e outputs)" if not bad
                  else f"MISMATCH on ranks {bad}",
                  "binomial_scatter_1GiB": "bit-exact vs oracle on every rank" if not bad_sc
                  else f"MISMATCH on ranks {bad_sc}"}
        cpu_base = {"value": round(4 * n / t_cpu / 1e9, 5), "unit": "GB/s", "cores": thr, "kind": "port",
                    "sample": f"full cfg2: {world} ranks x 512 MiB ring allreduce simulated on the host, one step",
                    "cpu": cpu_model()}
        ok = not bad and not bad_sc
    else:
        ok = True
    flag = [None] * world
    dist.all_gather_object(flag, ok)

    value = S_CFG2 / t
    peak, peak_kind = peaks()
    if rank == 0:
        line = _line(
            world, args.steps, warm, round(value / 1e9, 2), round(t * 1e3, 4), shared_config(world),
            detail={"value_is": "uncompressed bytes per rank / max-over-ranks device time of one allreduce",
                    "nccl_allreduce_gbs": nccl_gbs, "compression_ratio": cr,
                    "collective_roofline_gbs": round(900.0 * (cr or 1.0), 1),
                    "collective_roofline_frac": round(value / 1e9 / (900.0 * (cr or 1.0)), 4),
                    "scatter_1GiB_gbs": round(scatter_gbs, 2), "nccl_scatter_1GiB_gbs": nccl_scatter_gbs,
                    "rd_allreduce_gbs": round(rd_gbs, 2)},
            roofline={"bound": "hbm", "kernel": "fused RS step (k_tile_encode<STEP>, slotted output)",
                      "achieved": round(step_gbs, 1), "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                      "frac": round(step_gbs / peak, 4), "traffic": _traffic(f"fused_step_peer_{m}"),
                      "algorithmic_bytes_per_launch": int(step_bytes), "avg_step_us": round(t_step * 1e6, 2),
                      "bytes_per_unit": "4 B local + received and produced compressed bytes per value"},
            cpu_baseline=cpu_base,
            e2e={"value": round(S_CFG2 / t_e2e / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                 "d2h_bytes_per_step": 4 * n,
                 "api": "pinned host f32 -> H2D -> Communicator.ring_allreduce -> D2H, consecutive steps pipelined "
                        "on 3 streams, max over ranks"},
            gpu_launches=launches, clocks=clk.summary(), parity=parity)
        if oversub:
            line["rehearsal"] = (f"{world} ranks on {torch.cuda.device_count()} GPUs (time-sliced): "
                                 "code-path check, not a measurement")
        print(json.dumps(line), flush=True)
    c.close()
    dist.barrier()
    dist.destroy_process_group()
    if not all(flag):
        print("parity failure", file=sys.stderr)
        return 1
    return 0


# ---------------------------------------------------------------------------
# configs[3]: message-size sweep (N > 1)
# ---------------------------------------------------------------------------


def bench_sweep(args):
    import math

    import torch
    import torch.distributed as dist

    from paper_2308_05199_b200 import comm

    rank, world, local, dev, oversub = _init_dist()
    c = comm.Communicator(dist.group.WORLD, dev)
    s = torch.cuda.current_stream()
    mib = 1
    while mib <= args.sweep_max_mib:
        n = mib << 18
        i = torch.arange(n, dtype=torch.float64, device=dev)
        ph = 0.37 * rank
        x = (0.5 * torch.sin(2 * math.pi * i / 65536 + ph) + 0.25 * torch.sin(2 * math.pi * i / 4099 + ph)).float()
        del i
        out = torch.empty_like(x)
        tn = None
        if not oversub:
            y = x.clone()
            for _ in range(2):
                dist.all_reduce(y)
            tn = _timed_calls(lambda: dist.all_reduce(y), s, 7, dev)
            del y
        for eb in (1e-2, 1e-3, 1e-4):
            for _ in range(2):
                c.ring_allreduce(x, eb, out=out, check=False)
            t = _timed_calls(lambda: c.ring_allreduce(x, eb, out=out, check=False), s, 7, dev)
            c.check()
            cr = c.compression_ratio()
            if rank == 0:
                cfg = {"workload": f"ring-allreduce sweep point, {mib} MiB f32 per rank, eb={eb:g}",
                       "bytes_per_rank": 4 * n, "eb": eb, "ranks": world, "l2": "median of 7 calls"}
                print(json.dumps(_line(world, 7, 2, round(4 * n / t / 1e9, 2), round(t * 1e3, 4), cfg,
                                       detail={"compression_ratio": cr,
                                               "nccl_allreduce_gbs": round(4 * n / tn / 1e9, 2) if tn else None,
                                               "ratio_vs_nccl": round(tn / t, 3) if tn else None})), flush=True)
        del x, out
        torch.cuda.empty_cache()
        mib *= 2
    c.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweep", action="store_true", help="configs[3]: allreduce message-size sweep (N > 1)")
    ap.add_argument("--sweep-max-mib", type=int, default=2048)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.sweep:
        return bench_sweep(args)
    if args.gpus <= 1 and world <= 1:
        return bench_codec(args)
    return bench_allreduce(args)


if __name__ == "__main__":
    sys.exit(main())
