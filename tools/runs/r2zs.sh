set -u
# chunk-minor task order (shift / mask locate) for several chunks: S = 128, 256, 1024
O=gpurun_out/r2zs; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "batch or view or c4" > $O/pytest.txt 2>&1
for S in 128 256 1024; do
for lib in prev ""; do
echo "== ${lib:-chunk-minor} S=$S" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 600 python tools/env_ab.py --config C4 --S $S --reps 3 --var "" >> $O/ab.txt 2>&1
done; done
echo done
