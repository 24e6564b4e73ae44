set -u
# group wait of partials only in the single-chunk kernels (multi-chunk kernels back to the per-partial wait)
O=gpurun_out/r2zz3; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
for S in 128 256 1024 64; do
for lib in prev ""; do
echo "== ${lib:-onechunk-group} S=$S" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 600 python tools/env_ab.py --config C4 --S $S --reps 3 --var "" >> $O/ab.txt 2>&1
done; done
echo done
