"""Turn gpurun_out/prof/ (tools/make_profiles.sh) into committed profiles/ text files."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles"
TAG = sys.argv[3] if len(sys.argv) > 3 else "round1"
os.makedirs(DST, exist_ok=True)

for name in ("launches_summary.txt", "syncbench.txt", "prop_sweep_C3.txt", "prop_sweep_C5.txt",
             "trace_C3.txt", "kahn_C3.txt", "gpu.txt"):
    p = os.path.join(SRC, name)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(DST, f"{TAG}_{name}"))

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__block_size", "smsp__inst_executed.sum"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        out.append(d)
    return out


traffic = {}
for rep, label in (("propagate.ncu-rep", "propagate"), ("kahn.ncu-rep", "kahn")):
    p = os.path.join(SRC, rep)
    if not os.path.exists(p):
        continue
    rows = raw(p)
    lines = [f"# ncu --set full --clock-control none ({label}); bench.py --ncu (C4, S=64)"]
    for d in rows:
        lines.append(json.dumps(d))
    stalls = subprocess.run([sys.executable, "tools/ncu_stalls.py", p, ".", "15"],
                            capture_output=True, text=True).stdout
    lines.append("\n# top stalled SASS instructions (warp-state samples)\n" + stalls)
    with open(os.path.join(DST, f"{TAG}_ncu_{label}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if label == "propagate":
        tot = 0.0
        for d in rows:
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = d[m].split()
                v = float(v.replace(",", ""))
                tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic["C4"] = tot
if traffic:
    with open(os.path.join(DST, "traffic.json"), "w") as f:
        json.dump({"C4": traffic["C4"], "what": "dram__bytes_read.sum + dram__bytes_write.sum of "
                   "the forward + backward propagation kernels of one C4 step (ncu --set full)"},
                  f, indent=1)
print("ok", os.listdir(DST))
