"""Selected raw metrics per kernel from an ncu report.

    python tools/ncu_metrics.py report.ncu-rep [regex ...]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pats = sys.argv[2:] or [r"dram__bytes_(read|write)\.sum$", r"lts__t_sector_hit_rate", r"lts__t_sectors_srcunit_tex_op_read\.sum$",
                        r"lts__throughput", r"sm__warps_active", r"smsp__inst_executed\.sum$", r"gpu__time_duration\.sum$",
                        r"l1tex__t_requests_pipe_lsu_mem_global_op_ld\.sum$", r"l1tex__t_sectors_pipe_lsu_mem_global_op_ld\.sum$",
                        r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$", r"smsp__average_warp", r"dram__throughput",
                        r"l1tex__throughput", r"lts__t_sectors_op_read\.sum$", r"lts__t_sectors_op_write\.sum$",
                        r"lts__t_sectors_lookup_miss\.sum$", r"l1tex__m_xbar2l1tex_read_bytes", r"sm__throughput"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:100])
    for i, h in enumerate(hdr):
        if any(re.search(p, h) for p in pats):
            print(f"    {h:70s} {r[i]:>20s} {units[i]}")
