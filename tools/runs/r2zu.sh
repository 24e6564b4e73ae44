set -u
O=gpurun_out/r2zu; mkdir -p $O
HF_PROP_TIMES=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/stages.txt 2>&1
HF_PROP_TIMES=1 HF_PREFILL=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/stages_prefill.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv \
    python bench.py --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary > /dev/null 2>&1
python tools/launches.py $O/launches_C4.csv > $O/launches_C4_summary.txt 2>&1
echo done
