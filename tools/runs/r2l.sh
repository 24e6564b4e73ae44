set -u
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE2=0 --var HF_WIDE2=0,HF_L2_PERSIST=1 --var HF_WIDE2=1 --var HF_WIDE2=1,HF_L2_PERSIST=1 > $O/ab_c5.txt 2>&1
nvidia-smi -q | grep -i -A3 "L2\|persist" | head -20 > $O/smi.txt
echo done
