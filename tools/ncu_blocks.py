"""Hot SASS basic blocks of one ncu report with per-reason stall samples, each
block labelled with the CUDA source line of its first instruction (needs
-lineinfo + --import-source):  python tools/ncu_blocks.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, cur, ins = None, "", []
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10:
        continue
    if r[0]:
        cur = f"L{r[0]}: {r[1].strip()[:70]}"
        continue
    if r[2] == "...":
        continue
    try:
        n = float(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                st[h[6:]] = float(r[i])
            except ValueError:
                pass
    ins.append((int(r[2], 16), r[3].strip(), n, st, cur))
ins.sort(key=lambda x: x[0])
blocks, b = [], None
for a, s, n, st, src in ins:
    if b is None or n != b["n"]:
        b = {"n": n, "ins": [], "st": {}, "src": src, "a": a}
        blocks.append(b)
    b["ins"].append(s)
    for k, v in st.items():
        b["st"][k] = b["st"].get(k, 0) + v
tot = sum(x["n"] * len(x["ins"]) for x in blocks) or 1
stot = sum(sum(x["st"].values()) for x in blocks) or 1
blocks.sort(key=lambda x: -x["n"] * len(x["ins"]))
for x in blocks[:top]:
    ops = {}
    for s in x["ins"]:
        w = s.split()
        op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    topops = " ".join(f"{k}{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    stl = " ".join(f"{k}{100 * v / stot:.1f}" for k, v in sorted(x["st"].items(), key=lambda kv: -kv[1])[:4] if v > 0)
    print(f"{100 * x['n'] * len(x['ins']) / tot:5.1f}% n={x['n']:.3g} len={len(x['ins'])} [{topops}] stalls: {stl}\n       {x['src']}")
