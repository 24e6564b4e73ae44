set -u
# last knobs with the final code: poll back-off cap, sentinel fill grid
O=gpurun_out/r2zz16; mkdir -p $O
for rep in 1 2; do
timeout 900 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" --var HF_SLEEP_MAX=48 --var HF_SLEEP_MAX=96 --var HF_SLEEP_MAX_B=48 --var HF_FILL_CTAS=3552 --var HF_FILL_CTAS=4736 >> $O/ab.txt 2>&1
done
echo done
