set -u
# task-count gate (HF_GATE_LEVELS16 = lag in 1/16 levels of tasks; 0 = off)
O=gpurun_out/r2zz5; mkdir -p $O
L=$PWD/paper_2203_08395_b200
HF_GATE_LEVELS16=16 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "batch or tiny or golden or c4" > $O/pytest.txt 2>&1
for rep in 1 2; do
echo "== prev" >> $O/ab.txt
HF_LIB=$L/libhf_prev.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" >> $O/ab.txt 2>&1
echo "== gate build" >> $O/ab.txt
timeout 900 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" --var HF_GATE_LEVELS16=8 --var HF_GATE_LEVELS16=16 --var HF_GATE_LEVELS16=24 --var HF_GATE_LEVELS16=32 --var HF_GATE_LEVELS16=16,HF_GATE_SLEEP=256 >> $O/ab.txt 2>&1
done
echo done
