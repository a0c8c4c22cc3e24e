"""Attribute executed warp instructions and stall samples of one ncu report to
CUDA source lines (needs -lineinfo):  python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, cur, agg = None, None, None, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) // 2:
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:100])
            continue
        try:
            n = float(r[hdr.index("Instructions Executed")])
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += n
        a[1] += s
    tot = sum(v[0] for v in agg.values()) or 1
    stot = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.4g}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / tot:5.1f}%  stall {100 * v[1] / stot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
