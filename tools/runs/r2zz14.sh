set -u
# forward task weight at four and more chunks (S = 256 / 512 / 1024): 20 (default) vs 24 / 28
O=gpurun_out/r2zz14; mkdir -p $O
timeout 900 python tools/env_ab.py --config C4 --S 256 --reps 3 --var "" --var HF_TW_F=24 --var HF_TW_F=28 >> $O/ab.txt 2>&1
timeout 900 python tools/env_ab.py --config C4 --S 1024 --reps 3 --var "" --var HF_TW_F=24 --var HF_TW_F=28 >> $O/ab.txt 2>&1
echo done
