"""One-line stall / issue summary of ncu reports: python tools/ncu_stalls.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    parts = []
    for a, b in zip(h, v):
        short = a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
        if a in KEYS:
            parts.append(f"{short.split('.')[0]}={b}")
        elif "stall" in a and a.endswith("_per_issue_active.ratio") and "not_issued" not in a:
            try:
                if float(b) > 0.05:
                    parts.append(f"{short}={float(b):.2f}")
            except ValueError:
                pass
    print(rep.split("/")[-1], " ".join(parts))
