"""Print the bench lines of gpurun_out/ab/bench.txt (tools/ab.sh) side by side."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab/bench.txt"
tag = None
for line in open(path):
    if line.startswith("=="):
        tag = line[3:].strip()
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    ph = d.get("phases_ms", {})
    print(f"{tag:12s} {d['value'] / 1e9:7.2f} G  {d['ms_per_step']:.3f} ms  frac {d['roofline']['frac']:.3f}  "
          + "  ".join(f"{k} {v:.3f}" for k, v in ph.items()))
