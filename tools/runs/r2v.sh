set -u
O=gpurun_out/r2v; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide3 -c 2 -o $O/wide3 python bench.py --config C5 --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/wide3.ncu-rep > $O/sum.txt 2>&1
python tools/ncu_stalls.py $O/wide3.ncu-rep k_wide3 30 > $O/stalls.txt 2>&1
ncu -i $O/wide3.ncu-rep --page details --csv > $O/details.csv 2>&1
echo done
