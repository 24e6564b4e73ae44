set -u
O=gpurun_out/r2e; mkdir -p $O
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" --var HF_CTAS_PER_SM=6 --var HF_CTAS_PER_SM=5 --var HF_CTAS_PER_SM=4 --var HF_CTAS_PER_SM=3 > $O/ab_cap64.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 8 --reps 5 --var "" --var HF_CTAS_PER_SM=5 --var HF_CTAS_PER_SM=4 --var HF_CTAS_PER_SM=3 --var HF_CTAS_PER_SM=2 > $O/ab_cap8.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide1 -c 2 -o $O/wide1 python bench.py --config C5 --ncu --steps 1 --warmup 0 > $O/ncu_wide.log 2>&1
python tools/ncu_summary.py $O/wide1.ncu-rep > $O/ncu_wide1_summary.txt 2>&1
python tools/ncu_lines.py $O/wide1.ncu-rep k_wide1 40 > $O/ncu_wide1_lines.txt 2>&1
python tools/ncu_stalls.py $O/wide1.ncu-rep k_wide1 25 > $O/ncu_wide1_stalls.txt 2>&1
echo done
