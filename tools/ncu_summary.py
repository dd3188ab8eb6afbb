"""Summarise an ncu --set full report (raw page) into a small text table for profiles/."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for r in rows[2:]:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {r[i][:90]} {units[i]}")
    st = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(float(r[h.index(k)] or 0) for k in st) or 1.0
    top = sorted(((float(r[h.index(k)] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in st), reverse=True)[:6]
    print("stall samples (share):", ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in top))
    print("-" * 100)
