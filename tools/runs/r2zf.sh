set -u
# level gate (HF_GATE_LAG): parity with the gate on, A/B against the previous kernel
O=gpurun_out/r2zf; mkdir -p $O
L=$PWD/paper_2203_08395_b200
HF_LIB=$L/libhf_mb.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "batch or tiny or golden" > $O/pytest_mb.txt 2>&1
for rep in 1 2; do
echo "== base" >> $O/ab.txt
HF_LIB=$L/libhf_base.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
echo "== mb (launch bounds 7/5)" >> $O/ab.txt
HF_LIB=$L/libhf_mb.so timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var HF_GATE_LAG=0 --var HF_GATE_LAG=1 --var HF_GATE_LAG=2 --var HF_GATE_LAG=3 --var HF_GATE_LAG=2,HF_GATE_SLEEP=1024 >> $O/ab.txt 2>&1
echo "== default build (128/80 regs)" >> $O/ab.txt
HF_LIB=$L/libhf.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var HF_GATE_LAG=0 --var HF_GATE_LAG=2 >> $O/ab.txt 2>&1
done
echo done
