"""Per-source-line instruction counts and stall samples of one kernel, joining an
ncu report's per-SASS counters (source page) with nvdisasm's line table of the same
build (ncu's own CUDA-source view needs the source on the profiling box).

    cuobjdump -xelf all paper_2203_08395_b200/libhf.so   # in a scratch dir
    nvdisasm -g -c --print-line-info propagate.sm_100a.cubin > prop.sass
    python tools/ncu_srcmap.py report.ncu-rep prop.sass '<kernel regex>' [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def line_table(sass_file, mangled):
    """offset -> (file, line) for the function whose section name contains `mangled`."""
    out, cur, on = {}, None, False
    for ln in open(sass_file):
        if ln.startswith("//------") and ".text." in ln:
            on = mangled in ln
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, sass, pat = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    for blk in re.split(r'(?m)^"Kernel Name",', txt)[1:]:
        name = blk.split("\n", 1)[0]
        if not re.search(pat, name):
            continue
        rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
        h = rows[0]
        ia, ii, iss = h.index("Address"), h.index("Instructions Executed"), h.index(
            "Warp Stall Sampling (All Samples)")
        data = []
        for r in rows[1:]:
            if len(r) < len(h):
                continue
            try:
                data.append((int(r[ia], 16), float(r[ii] or 0), float(r[iss] or 0)))
            except ValueError:
                pass
        base = data[0][0]
        # the mangled name of this instantiation: find the section whose offsets match
        secs = re.findall(r"\.text\.(\S+k_flow\S+) -", open(sass).read())
        best = None
        for sec in secs:
            tab = line_table(sass, sec)
            if len(tab) == len(data):
                tpl = re.search(r"k_flow<([^>]*)>", name).group(1).replace("(int)", "").replace(
                    "(bool)", "").replace(" ", "").split(",")
                enc = "".join(("Li%sE" % x) if i < 2 else ("Lb%sE" % x) for i, x in enumerate(tpl))
                if enc in sec:
                    best = tab
                    break
        if best is None:
            print("no matching section for", name[:90])
            continue
        src = {}
        agg = collections.defaultdict(lambda: [0.0, 0.0])
        for a, i, s in data:
            key = best.get(a - base, ("?", 0))
            agg[key][0] += i
            agg[key][1] += s
        ti = sum(v[0] for v in agg.values()) or 1
        ts = sum(v[1] for v in agg.values()) or 1
        lines = {}
        try:
            lines = dict(enumerate(open("paper_2203_08395_b200/csrc/" + "propagate.cu").read().split("\n"), 1))
        except OSError:
            pass
        print(f"== {name[:110]}\n   instructions {ti:.3e}, stall samples {ts:.0f}")
        for (f, l), (i, s) in sorted(agg.items(), key=lambda kv: -(kv[1][0] / ti + kv[1][1] / ts))[:top]:
            text = lines.get(l, "").strip() if f == "propagate.cu" else ""
            print(f"   {100 * i / ti:5.1f}% {100 * s / ts:5.1f}%  {f}:{l:<5} {text[:80]}")


if __name__ == "__main__":
    main()
