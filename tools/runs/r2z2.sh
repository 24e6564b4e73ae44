set -u
O=gpurun_out/r2z2; mkdir -p $O
L=$PWD/paper_2203_08395_b200/libhf_pe16.so
HF_LIB=$L timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_TW=8 --var HF_TW=10 --var HF_TW=12 > $O/ab_tw_pe16.txt 2>&1
HF_LIB=$L timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 120 -k "batch_small or tiny" > $O/pytest_pe16.txt 2>&1
echo done
