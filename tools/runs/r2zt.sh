set -u
# phase: forward NaN-prefill of rat (HF_PREFILL=1) and fill grid sizes, with the faster kernels
O=gpurun_out/r2zt; mkdir -p $O
for rep in 1 2; do
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_PREFILL=1 --var HF_FILL_CTAS=296 --var HF_FILL_CTAS=2368 >> $O/ab.txt 2>&1
done
echo done
