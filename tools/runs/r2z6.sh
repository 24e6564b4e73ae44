set -u
O=gpurun_out/r2z6; mkdir -p $O
timeout 900 python tools/env_ab.py --config C4 --S 64 --reps 9 --var "" --var HF_TW_F=9 --var HF_TW_F=10 --var HF_TW_F=11 --var HF_TW_B=9 --var HF_TW_B=10 --var HF_TW_B=11 --var HF_TW_B=12 > $O/ab_tw.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 8 --reps 7 --var "" --var HF_TW=16 --var HF_TW=24 > $O/ab_tw8.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 256 --reps 5 --var "" --var HF_TW=8 --var HF_TW=10 > $O/ab_tw256.txt 2>&1
echo done
