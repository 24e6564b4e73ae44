set -u
# Kahn append: cooperative only when a lane has more than 4 entries (hybrid) vs always vs never
O=gpurun_out/r2zz18; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "golden or levelize or cycle or C2 or full_c3 or tiny or C5" > $O/pytest.txt 2>&1
for rep in 1 2; do
for lib in seq coop ""; do
for c in C3 C2-random C5; do
echo "== ${lib:-hybrid} $c" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so HF_LEV_TIMES=1 timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary 2>&1 | grep -E "levelize stages" | tail -1 >> $O/ab.txt
done; done; done
echo done
