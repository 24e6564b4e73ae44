set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python tools/env_ab.py --config C4 --graph C3 --S 64 --reps 5 --var "" --var HF_SC=32 --var HF_SC=16 --var HF_SC=32,HF_TW=16 --var HF_SC=16,HF_TW=24 --var HF_SLEEP_MAX=32 --var HF_SLEEP_MAX=128 > $O/ab_sc.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --graph C3 --S 8 --reps 5 --var "" --var HF_TW=16 --var HF_TW=24 --var HF_CONCURRENT=1 --var HF_SLEEP_MAX=32 > $O/ab_s8.txt 2>&1
echo done
