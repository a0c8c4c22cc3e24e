"""Summarise an ncu --set full report (.ncu-rep) into JSON: key throughput metrics +
executed-SASS opcode mix.  Usage: python tools/ncu_summary.py report.ncu-rep [label]"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def summarise(rep, label=None):
    rows = list(csv.reader(run([rep, "--page", "raw", "--csv"]).splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    out = {"report": rep, "label": label, "kernel": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            out[k] = {"value": v[h.index(k)], "unit": units[h.index(k)]}
    srows = list(csv.reader(run([rep, "--page", "source", "--csv", "--print-source", "sass"]).splitlines()))
    hh = srows[1]
    iE, iS = hh.index("Instructions Executed"), hh.index("Source")
    c = collections.Counter()
    tot = 0
    for r in srows[2:]:
        try:
            e = int(r[iE] or 0)
        except (ValueError, IndexError):
            continue
        s = r[iS].strip()
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        op = op.split(".")[0]
        c[op] += e
        tot += e
    out["warp_instructions"] = tot
    out["opcode_mix_pct"] = {k: round(100 * n / tot, 2) for k, n in c.most_common(16)}
    return out


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None), indent=1))
