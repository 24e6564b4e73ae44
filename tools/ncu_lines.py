"""Per CUDA-source-line instruction counts and stall samples from an ncu report
(source page, --import-source on captures), per kernel: where a kernel's issue
slots and stalls go.

    python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import re
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', txt)
    for blk in blocks[1:]:
        name = blk.split("\n", 1)[0]
        if not re.search(pat, name):
            continue
        rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
        hdr = rows[0]
        def col(*names):
            for nm in names:
                if nm in hdr:
                    return hdr.index(nm)
            return None
        ci = col("Instructions Executed", "Warp Instructions Executed")
        cs = col("Warp Stall Sampling (All Samples)")
        cl = col("#", "Line", "# Line")
        csrc = col("Source")
        data = []
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            data.append((num(r[ci]) if ci is not None else 0, num(r[cs]) if cs is not None else 0,
                         r[cl] if cl is not None else "", r[csrc] if csrc is not None else ""))
        ti = sum(d[0] for d in data) or 1
        ts = sum(d[1] for d in data) or 1
        print(f"== {name[:110]}\n   instructions {ti:.3e}, stall samples {ts:.0f}")
        print(f"   {'inst%':>6} {'stall%':>6}  line  source")
        for i, s, ln, src in sorted(data, key=lambda d: -(d[0] / ti + d[1] / ts))[:top]:
            print(f"   {100 * i / ti:6.1f} {100 * s / ts:6.1f}  {ln:>5}  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
