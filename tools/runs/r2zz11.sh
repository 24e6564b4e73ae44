set -u
# task weight re-tune at S = 64 after the late k_flow changes
O=gpurun_out/r2zz11; mkdir -p $O
for rep in 1 2; do
timeout 900 python tools/env_ab.py --config C4 --S 64 --reps 5 --var HF_TW_F=10 --var HF_TW_F=9 --var HF_TW_F=8 --var HF_TW_F=7 >> $O/ab.txt 2>&1
done
echo done
