set -u
O=gpurun_out/r2z9; mkdir -p $O
for rep in 1 2; do
for v in "" sp6 sp10 sp12; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-sp8}" >> $O/ab.txt
  HF_LIB=$lib timeout 200 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
HF_LIB=$PWD/paper_2203_08395_b200/libhf_sp12.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 120 -k "batch_small or tiny or multi_edges" > $O/pytest_sp12.txt 2>&1
echo done
