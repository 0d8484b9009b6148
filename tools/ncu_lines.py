"""Aggregate an ncu source page (--print-source cuda,sass --csv) per source line.
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys, io, os
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = []
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = os.path.basename(r[1]); continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        rows.append((f, int(r[0]), r[1].strip()[:80], int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0)))
    except (ValueError, KeyError):
        pass
tot_i = sum(x[3] for x in rows) or 1
tot_s = sum(x[4] for x in rows) or 1
print(f"total inst {tot_i}  samples {tot_s}")
for key, name in ((3, "instructions"), (4, "stall samples")):
    print(f"--- top by {name}")
    for x in sorted(rows, key=lambda x: -x[key])[:top]:
        print(f"{x[0]:>14s}:{x[1]:<5d} inst {100*x[3]/tot_i:5.1f}%  samp {100*x[4]/tot_s:5.1f}%  {x[2]}")
