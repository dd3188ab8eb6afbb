"""Hot CUDA source lines of one kernel from an ncu report (warp-stall samples aggregated per
line, top stall reasons): python tools/ncu_hot.py rep.ncu-rep [N]"""
import collections
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = "?", None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1].strip()
    for i, h in enumerate(hdr):
        if i >= 4 and (h == "Warp Stall Sampling (All Samples)" or (h.startswith("stall_") and "Not Issued" not in h)):
            try:
                agg[key][h] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(c["Warp Stall Sampling (All Samples)"] for c in agg.values()) or 1.0
top = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:n]
for (f, ln), c in top:
    s = c["Warp Stall Sampling (All Samples)"]
    st = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} {src[(f, ln)][:64]:64s} " + " ".join(f"{k}={v:.0f}" for v, k in st if v))
