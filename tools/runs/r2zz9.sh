set -u
# k_wide3 registers: neighbour keys lane-distributed (79 -> 63 registers, 4 CTAs/SM), units per warp
O=gpurun_out/r2zz9; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
HF_LIB=$L/libhf_u10.so timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 600 > $O/pytest_u10.txt 2>&1
for rep in 1 2; do
for lib in prev "" u10 u6; do
echo "== ${lib:-keys-packed U8}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C5 --single --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
echo done
