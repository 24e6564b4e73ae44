set -u
O=gpurun_out/r2za; mkdir -p $O
timeout 900 python tools/env_ab.py --config C4 --S 256 --reps 5 --var "" --var HF_TW_F=14,HF_TW_B=16 --var HF_TW_F=16,HF_TW_B=18 --var HF_TW_F=20,HF_TW_B=22 > $O/ab256.txt 2>&1
timeout 900 python tools/env_ab.py --config C4 --S 1024 --reps 3 --var "" --var HF_TW_F=16,HF_TW_B=18 --var HF_TW_F=20,HF_TW_B=22 > $O/ab1024.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 128 --reps 5 --var "" --var HF_TW_F=11,HF_TW_B=10 --var HF_TW_F=16,HF_TW_B=18 > $O/ab128.txt 2>&1
echo done
