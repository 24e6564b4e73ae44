set -u
O=gpurun_out/r2n; mkdir -p $O
L=$PWD/paper_2203_08395_b200/libhf_idx.so
HF_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "batch or tiny or config_single or early or critical" > $O/pytest_idx.txt 2>&1
for S in 64 8 1; do
for v in "" idx; do
  lib=""; [ -n "$v" ] && lib=$L
  echo "== ${v:-default} S=$S" >> $O/ab.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C4 --S $S --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
