set -u
# locate fast path for one scenario chunk (nch == 1): parity subset + A/B
O=gpurun_out/r2zh; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "batch or tiny or golden or c4" > $O/pytest.txt 2>&1
for rep in 1 2; do
for lib in base ""; do
echo "== ${lib:-new}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
