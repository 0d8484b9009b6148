"""Instructions per tile by source region from an ncu source page.
python tools/ncu_regions.py report.ncu-rep ntiles"""
import csv, subprocess, sys, io, os, collections
rep, ntiles = sys.argv[1], int(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None; hdr = None; acc = collections.Counter(); samp = collections.Counter(); lines = collections.defaultdict(list)
import re
def _dev_regions():
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_05199_b200", "csrc", "gz_device.cuh")).read().splitlines()
    find = lambda pat: next(i + 1 for i, l in enumerate(src) if re.search(pat, l))
    fb, lc, ap, lr = find(r"int fast_block\("), find(r"void load_codes\("), find(r"^struct Appender"), find(r"void load_row\(")
    return [(fb - 12, lc - 2, "fast_block"), (lc - 1, ap - 1, "codes ld/st"), (ap, lr - 1, "appender"), (lr, lr + 11, "load_row"), (90, fb - 13, "slow")]
REG = {"gz_device.cuh": _dev_regions(),
       "gz_codec.cu": [(412, 438, "enc: step decode"), (439, 481, "enc: quantise/size"), (482, 491, "enc: scan"), (492, 555, "enc: pack"), (556, 560, "enc: sidecar"),
                       (365, 396, "prefetch"), (397, 411, "reload"), (328, 351, "geom"), (572, 731, "kernel loop/claim"), (175, 190, "stage"), (199, 320, "decode"), (733, 918, "gather")]}
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "File Path": f = os.path.basename(r[1]); continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ln, ins, s = int(r[0]), int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0)
    except (ValueError, KeyError):
        continue
    name = "other:" + f
    for a, b, nm in REG.get(f, []):
        if a <= ln <= b: name = nm; break
    acc[name] += ins; samp[name] += s
tot = sum(acc.values()); ts = sum(samp.values()) or 1
print("total instr/tile %.0f" % (tot / ntiles))
for k, v in acc.most_common():
    print("%-22s %7.1f instr/tile  %5.1f%% samples" % (k, v / ntiles, 100 * samp[k] / ts))
