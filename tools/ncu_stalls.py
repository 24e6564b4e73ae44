"""Top stalled SASS instructions from an ncu report (source page), per kernel.

    python tools/ncu_stalls.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', txt)
    for blk in blocks[1:]:
        name = blk.split("\n", 1)[0]
        if not re.search(pat, name):
            continue
        rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
        hdr = rows[0]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = 0
        data = []
        for r in rows[1:]:
            if len(r) <= si:
                continue
            try:
                s = int(r[si])
            except ValueError:
                continue
            tot += s
            reasons = sorted(((int(r[c]) if r[c].isdigit() else 0, hdr[c][6:]) for c in cols),
                             reverse=True)[:3]
            data.append((s, r[0][-5:], r[1].strip(), reasons))
        print(f"== {name[:100]}  total samples {tot}")
        agg = {}
        for s, a, src, reasons in data:
            for v, k in reasons:
                agg[k] = agg.get(k, 0) + v
        for s, a, src, reasons in sorted(data, reverse=True)[:top]:
            rs = " ".join(f"{k}:{v}" for v, k in reasons if v)
            print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {a}  {src[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
