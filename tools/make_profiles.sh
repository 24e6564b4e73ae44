#!/bin/bash
# Run on the GPU box (gpurun): produce the round's evidence under gpurun_out/prof/.
#   launch list of one bench step, ncu --set full of the two propagation kernels
#   and the Kahn levelizer, S sweeps, per-task dataflow traces.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT/tr
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --ncu --steps 1 --warmup 0 > /dev/null 2>&1
python tools/launches.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 \
    -o $OUT/flow python bench.py --ncu --steps 1 --warmup 0 > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/flow.ncu-rep > $OUT/ncu_flow_summary.txt 2>&1
python tools/ncu_stalls.py $OUT/flow.ncu-rep k_flow 15 > $OUT/ncu_flow_stalls.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_lev_kahn -c 1 \
    -o $OUT/kahn python bench.py --ncu --steps 1 --warmup 0 > $OUT/ncu_kahn.log 2>&1
python tools/ncu_summary.py $OUT/kahn.ncu-rep > $OUT/ncu_kahn_summary.txt 2>&1
timeout 300 python tools/prop_sweep.py --S 1,4,16,64,256,1024 > $OUT/prop_sweep_C3.txt 2>&1
timeout 200 python tools/prop_sweep.py --config C5 --S 1,4 --reps 3 > $OUT/prop_sweep_C5.txt 2>&1
HF_TRACE=$OUT/tr/c3 timeout 100 python tools/prop_sweep.py --S 1,64 --reps 0 > /dev/null 2>&1
python tools/trace_report.py $OUT/tr/c3_fwd_S1.bin $OUT/tr/c3_bwd_S1.bin $OUT/tr/c3_fwd_S64.bin \
    $OUT/tr/c3_bwd_S64.bin > $OUT/trace_C3.txt 2>&1
python tools/kahn_report.py $OUT/tr/c3_kahn.bin > $OUT/kahn_C3.txt 2>&1
rm -f $OUT/tr/*.bin
# warm per-stage device times of the levelizer and the batch (CUDA events per stage)
HF_LEV_TIMES=1 HF_PROP_TIMES=1 timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 \
    | grep stages | tail -2 > $OUT/stages.txt
echo done
