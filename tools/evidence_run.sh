#!/bin/bash
# Round evidence on the GPU box: bench lines (3 runs), the reference arm, smoke(),
# the GPU tests, the NEXT-3 view sweep, MIS timing, then tools/make_profiles.sh.
set -u
mkdir -p gpurun_out/ev
for i in 1 2 3; do timeout 300 python bench.py > gpurun_out/ev/bench_$i.json 2>gpurun_out/ev/bench_$i.err; done
timeout 200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/ref.json 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/ev/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest.txt 2>&1
timeout 600 python tools/view_sweep.py > gpurun_out/ev/view_sweep.txt 2>&1
timeout 600 python tools/mis_time.py > gpurun_out/ev/mis.txt 2>&1
bash tools/make_profiles.sh
