set -u
O=gpurun_out/r2p; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 900 -k "batch or tiny or config_single or early or critical or top_k or multi_edges or isolated or hub or invalid or nonfinite or nan" > $O/pytest_lp1.txt 2>&1
HF_LIB=$PWD/paper_2203_08395_b200/libhf_f7b6.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "batch_small or full_c4 or multi_edges" > $O/pytest_f7b6.txt 2>&1
for S in 64 8; do
for v in lp0 "" f7 f7b6; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-lp1} S=$S" >> $O/ab.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C4 --S $S --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
