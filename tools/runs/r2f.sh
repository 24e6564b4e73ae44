set -u
O=gpurun_out/r2f; mkdir -p $O
for rep in 1 2; do
for v in "" nu3 nu4; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-default}" >> $O/ab_c5.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C5 --single --reps 5 --var "" >> $O/ab_c5.txt 2>&1
done; done
echo done
