set -u
# idle fill: the forward's warps NaN-fill rat while they wait (no separate rat fill)
O=gpurun_out/r2zv; mkdir -p $O
L=$PWD/paper_2203_08395_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 600 > $O/pytest.txt 2>&1
for rep in 1 2; do
echo "== prev" >> $O/ab.txt
HF_LIB=$L/libhf_prev.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
echo "== idle fill build" >> $O/ab.txt
timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_IDLE_FILL=0 >> $O/ab.txt 2>&1
done
for S in 256 16; do
timeout 600 python tools/env_ab.py --config C4 --S $S --reps 3 --var "" --var HF_IDLE_FILL=0 >> $O/ab.txt 2>&1
done
HF_PROP_TIMES=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > $O/stages.txt 2>&1
echo done
