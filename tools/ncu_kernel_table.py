"""Markdown table of the headline metrics of one-kernel ncu --set full reports.
python tools/ncu_kernel_table.py name=report.ncu-rep [name=report ...]"""
import csv
import io
import subprocess
import sys

METRICS = [("duration (µs)", "gpu__time_duration.sum", None),
           ("grid × block", None, None),
           ("registers / thread", "launch__registers_per_thread", None),
           ("warp-instructions (M)", "smsp__inst_executed.sum", 1e-6),
           ("issue active (%)", "smsp__issue_active.avg.pct_of_peak_sustained_active", None),
           ("warps active (% of 64)", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
           ("SM active cycles / elapsed (%)", None, None),
           ("DRAM read (MB)", "dram__bytes_read.sum", None),
           ("DRAM write (MB)", "dram__bytes_write.sum", None),
           ("L2 hit rate (%)", "lts__t_sector_hit_rate.pct", None)]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (x, u) for k, u, x in zip(h, units, v)}


def num(d, k):
    x, u = d[k]
    x = float(x.replace(",", ""))
    if k == "gpu__time_duration.sum":  # -> microseconds
        return x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    if u in ("Kbyte",):
        x *= 1e-3
    if u in ("Gbyte",):
        x *= 1e3
    if u == "byte":
        x *= 1e-6
    return x


cols = []
for arg in sys.argv[1:]:
    name, rep = arg.split("=", 1)
    d = raw(rep)
    col = []
    for label, key, scale in METRICS:
        if label == "grid × block":
            col.append(f"{d['launch__grid_size'][0]} × {d['launch__block_size'][0]}")
        elif label.startswith("SM active"):
            el = num(d, "gpc__cycles_elapsed.max") if "gpc__cycles_elapsed.max" in d else None
            act = num(d, "sm__cycles_active.avg")
            col.append(f"{100 * act / el:.0f}" if el else "")
        elif key in d:
            x = num(d, key)
            if scale:
                x *= scale
            col.append(f"{x:.2f}" if x < 1000 else f"{x:.0f}")
        else:
            col.append("")
    stalls = {k: float(v[0] or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    col.append(", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for k, v in top))
    cols.append((name, col))
print("| metric | " + " | ".join(n for n, _ in cols) + " |")
print("|---|" + "---|" * len(cols))
for i, (label, _, _) in enumerate(METRICS + [("top stall reasons (share of samples)", None, None)]):
    print(f"| {label} | " + " | ".join(c[i] for _, c in cols) + " |")
