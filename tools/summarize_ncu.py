"""Print the markdown summary rows used in profiles/ from gpu_round.sh outputs."""
import collections
import csv
import subprocess
import sys

launches = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_n1.csv"
rows = [l for l in open(launches) if l.startswith('"')]
r = list(csv.reader(rows))
h = r[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for x in r[1:]:
    v = float(x[vi].replace(",", ""))
    if x[ui] in ("nsecond", "ns"):
        v /= 1000
    agg[x[ki].split("(")[0].replace("void ", "")[:40]].append(v)
print("| kernel | launches | mean µs |\n|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} |")
want = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct"]
cols = {}
for name, f in (("k_tile_encode", "prof_bench_enc"), ("k_gather", "prof_bench_gather"), ("k_tile_decode", "prof_bench_dec")):
    out = subprocess.run(["ncu", "-i", f"gpurun_out/{f}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    hh, vv = rr[0], rr[2]
    d = {k: vv[hh.index(k)] for k in want if k in hh}
    st = []
    for i, k in enumerate(hh):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(vv[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    d["stalls"] = ", ".join(f"{n} {x:.2f}" for x, n in st[:3])
    cols[name] = d
print()
print("| metric | " + " | ".join(cols) + " |")
print("|---|" + "---|" * len(cols))
for k in want + ["stalls"]:
    print(f"| {k} | " + " | ".join(str(cols[c].get(k, "")) for c in cols) + " |")
