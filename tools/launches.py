"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        out.append((r[ki].split("(")[0].replace("void ", ""), v))
    return out


def summary(path):
    rows = load(path)
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v in rows:
        agg[k] += v
        cnt[k] += 1
    tot = sum(agg.values())
    lines = [f"{'total_us':>10} {'share':>6} {'n':>6} {'avg_us':>8}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"{v:10.1f} {v / tot:6.1%} {cnt[k]:6d} {v / cnt[k]:8.2f}  {k}")
    lines.append(f"{tot:10.1f} total over {len(rows)} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
