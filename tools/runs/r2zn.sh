set -u
# poll back-off cap with the cheap forward rounds
O=gpurun_out/r2zn; mkdir -p $O
timeout 900 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_SLEEP_MAX=32 --var HF_SLEEP_MAX=128 --var HF_SLEEP_MAX=256 --var HF_SLEEP_MAX=512 --var HF_SLEEP_MAX=1000 > $O/ab.txt 2>&1
timeout 900 python tools/env_ab.py --config C4 --S 8 --reps 5 --var "" --var HF_SLEEP_MAX=128 --var HF_SLEEP_MAX=256 >> $O/ab.txt 2>&1
echo done
