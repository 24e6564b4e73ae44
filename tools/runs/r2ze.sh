set -u
# where k_flow's issue slots go (C4, S = 64): per-source-line instructions + stalls
O=gpurun_out/r2ze; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 -o $O/flow_C4 \
    python bench.py --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_flow.log 2>&1
python tools/ncu_lines.py $O/flow_C4.ncu-rep k_flow 45 > $O/lines.txt 2>&1
python tools/ncu_stalls.py $O/flow_C4.ncu-rep k_flow 30 > $O/stalls.txt 2>&1
ncu -i $O/flow_C4.ncu-rep --page raw --csv > $O/raw.csv 2>&1
echo done
