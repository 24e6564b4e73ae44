set -u
# k_flow<..., ONE = true> (single scenario chunk): parity subset + A/B
O=gpurun_out/r2zi; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "batch or tiny or golden or c4" > $O/pytest.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 9 --var HF_ONE=1 --var HF_ONE=0 > $O/ab.txt 2>&1
timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 9 --var HF_ONE=1 --var HF_ONE=0 >> $O/ab.txt 2>&1
echo done
