set -u
O=gpurun_out/r2z5; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 120 -k "scratch_size or reuses_schedule" > $O/pytest.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_TW=6 --var HF_TW=8 --var HF_TW=10 > $O/ab_tw.txt 2>&1
echo done
