set -u
# edge-capped task schedule (k_tb_split): parity + A/B against the weight windows
O=gpurun_out/r2zd; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_EC=0 --var HF_TW_F=14,HF_TW_B=14 --var HF_TW=16 --var HF_TW=20 --var HF_EC=12 > $O/ab64.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 128 --reps 5 --var "" --var HF_EC=0 --var HF_TW=20 > $O/ab128.txt 2>&1
echo done
