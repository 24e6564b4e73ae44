set -u
# forward: vector R9 check of the delays (sum of d * 0) instead of per-element selects
O=gpurun_out/r2zw; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
for rep in 1 2; do
for lib in prev ""; do
echo "== ${lib:-vector-check}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
