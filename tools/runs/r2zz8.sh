set -u
# bitmask poll rounds in the single-chunk backward kernels too
O=gpurun_out/r2zz8; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
for rep in 1 2; do
for lib in prev ""; do
echo "== ${lib:-bwd-mask-one}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 8 --reps 5 --var "" >> $O/ab.txt 2>&1
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 32 --reps 5 --var "" >> $O/ab.txt 2>&1
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C3 --single --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
echo done
