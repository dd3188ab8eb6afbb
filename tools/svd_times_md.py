"""JSON lines of tools/svd_times.py -> the markdown table of profiles/svd_times_r02.md (round 1 values
from profiles/svd_times_r01.json in parentheses).  python tools/svd_times_md.py lines.jsonl [bench.json]"""
import json
import sys

rows = [json.loads(x) for x in open(sys.argv[1]) if x.startswith("{")]
old = {}
try:
    for r in json.load(open("profiles/svd_times_r01.json")):
        old[(r["config"], r["alg"], r["v"])] = r["svd_ms"]
except (OSError, ValueError, KeyError):
    pass
print("# Rank-k SVD time per view budget, all configs at full size (B200, round 2, end of round)\n")
print("`python tools/svd_times.py C1 C2 C3 C5` (one call, CUDA events, graph replay, median of reps, L2 flushed")
print("before each); C4 rows from the bench line (`profiles/bench_r02.json`, three concurrent calls per step).")
print("view roofline = sum over the views of max(A bytes / HBM, useful view flops / tensor peak).")
print("Round-1 times in parentheses.\n")
print("| config | dtype | alg | v | SVD ms | views/s | view-roofline ms | frac |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    o = old.get((r["config"], r["alg"], r["v"]))
    t = f"{r['svd_ms']:.3f}" + (f" ({o:.3f})" if o else "")
    print(f"| {r['config']} | {r['dtype']} | {r['alg']} | {r['v']} | {t} | {r['views_per_s']:.1f} | "
          f"{r['view_roofline_ms']:.3f} | {r['frac_of_view_roofline']:.3f} |")
if len(sys.argv) > 2:
    b = json.load(open(sys.argv[2]))
    for nm, ms in b["svd_ms"].items():
        rf = b["view_roofline_per_call"][nm]
        print(f"| C4 | f64 | {nm} | - | {ms:.1f} | - | {rf['roofline_ms']:.1f} | {rf['frac_of_view_roofline']:.3f} |")
