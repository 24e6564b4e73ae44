#!/bin/bash
# Final round-2 evidence on one B200 (after the late k_flow changes) (one gpurun call): GPU tests, smoke, one bench line per
# config (C4 three times), the NEXT-3 lines (S = 256, 1024 views), the reference arm,
# launch list of a C4 step, ncu --set full of the dominant kernels per config, the
# strong-scaling table and the view sweep.  Output: gpurun_out/ev2/
set -u
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.txt 2>&1
for i in 1 2 3; do timeout 400 python bench.py > $O/C4_$i.json 2> $O/C4_$i.err; done
for c in C1 C2-chain C2-tree C2-random C3 C5; do timeout 400 python bench.py --config $c > $O/$c.json 2> $O/$c.err; done
for s in 256 1024; do timeout 900 python bench.py --scenarios $s --no-secondary --no-e2e > $O/C4_S$s.json 2> $O/C4_S$s.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/C4.ref.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv \
    python bench.py --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
python tools/launches.py $O/launches_C4.csv > $O/launches_C4_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 -o $O/flow_C4 \
    python bench.py --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_flow.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide3 -c 2 -o $O/wide3_C5 \
    python bench.py --config C5 --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_wide.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lev_kahn -c 1 -o $O/kahn_C3 \
    python bench.py --config C3 --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_kahn.log 2>&1
for c in C2-chain C2-tree C2-random; do
  timeout 600 ncu --set full --clock-control none -k regex:"k_lev_" -c 6 -o $O/lev_$c \
      python bench.py --config $c --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_lev_$c.log 2>&1
done
for r in flow_C4 wide3_C5 kahn_C3 lev_C2-chain lev_C2-tree lev_C2-random; do
  python tools/ncu_summary.py $O/$r.ncu-rep > $O/ncu_${r}_summary.txt 2>&1
done
python tools/ncu_stalls.py $O/flow_C4.ncu-rep k_flow 15 > $O/ncu_flow_C4_stalls.txt 2>&1
timeout 600 python tools/strong_table.py > $O/strong_scaling.txt 2>&1
timeout 900 python tools/view_sweep.py > $O/view_sweep.txt 2>&1
HF_LEV_TIMES=1 HF_PROP_TIMES=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>&1 | grep stages | tail -2 > $O/stages.txt
HF_PROP_TIMES=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>&1 | grep "batch stages" | tail -2 >> $O/stages.txt
echo done > $O/done.txt
