set -u
O=gpurun_out/r2z; mkdir -p $O/tr
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_TW=8 --var HF_TW=9 --var HF_TW=10 --var HF_TW=16 > $O/ab_tw.txt 2>&1
echo done
