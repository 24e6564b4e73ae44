"""profiles/traffic.json from ncu --set full reports: DRAM bytes (read + write) per
launch of the dominant kernels, keyed "<config>/S<S>" as bench.py's roofline.traffic
looks them up.

    python tools/traffic_json.py C4/S64=report_C4.ncu-rep:k_flow C5/S1=report_C5.ncu-rep:k_wide3
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram_bytes(rep, pat):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for r in rows[2:]:
        if not re.search(pat, r[hdr.index("Kernel Name")]):
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i]) * scale[units[i]]
        out.append((r[hdr.index("Kernel Name")], tot))
    return out


def main():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[1:]:
        key, rest = arg.split("=", 1)
        rep, pat = rest.rsplit(":", 1)
        ks = dram_bytes(rep, pat)
        data[key] = {"traffic": sum(b for _, b in ks),
                     "per_kernel": {n[:80]: b for n, b in ks},
                     "source": f"ncu --set full, {os.path.basename(rep)} ({pat}): "
                               "dram__bytes_read.sum + dram__bytes_write.sum, one step"}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
