set -u
# ONE kernels for every one-chunk scenario count (S = 1, 2, 4..64)
O=gpurun_out/r2zr; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
for S in 8 16 32 1; do
timeout 300 python tools/env_ab.py --config C4 --S $S --reps 5 --var HF_ONE=1 --var HF_ONE=0 >> $O/ab.txt 2>&1
done
timeout 300 python tools/env_ab.py --config C3 --single --reps 5 --var HF_ONE=1 --var HF_ONE=0 >> $O/ab.txt 2>&1
echo done
