set -u
# task weight re-tune at S = 128 / 256 (several chunks)
O=gpurun_out/r2zz12; mkdir -p $O
timeout 900 python tools/env_ab.py --config C4 --S 128 --reps 3 --var "" --var HF_TW_F=10 --var HF_TW_F=14 --var HF_TW_B=12 --var HF_TW_B=16 >> $O/ab.txt 2>&1
timeout 900 python tools/env_ab.py --config C4 --S 256 --reps 3 --var "" --var HF_TW_F=16 --var HF_TW_F=24 --var HF_TW_B=12 --var HF_TW_B=16 >> $O/ab.txt 2>&1
echo done
