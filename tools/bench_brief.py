"""Print the key numbers of a bench.py JSON line (reads a log file)."""
import json
import sys

for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line)
        r = d.get("roofline") or {}
        print("ms/step", d.get("ms_per_step"), "value", d.get("value"), d.get("unit"))
        for k in ("forward_sweep", "adjoint_sweep"):
            if k in r:
                print(" ", k, r[k])
        if d.get("e2e"):
            print("  e2e", {k: d["e2e"][k] for k in ("value", "ms_per_step") if k in d["e2e"]})
        if d.get("cpu_baseline"):
            print("  cpu", d["cpu_baseline"])
        print("  clocks", d.get("clocks"))
