set -u
O=gpurun_out/r2q; mkdir -p $O
for S in 64 8; do
for v in lp0 "" f7 f7b6; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-lp1} S=$S" >> $O/ab.txt
  HF_LIB=$lib timeout 200 python tools/env_ab.py --config C4 --S $S --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
HF_WATCHDOG_MS=3000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 120 -k "batch or tiny or early or critical or top_k or multi_edges or isolated or invalid or nonfinite or nan" > $O/pytest_lp1.txt 2>&1
echo done
