set -u
O=gpurun_out/r2m; mkdir -p $O
for v in "" t512 t256; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-t1024}" >> $O/ab.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE2=0 --var HF_WIDE2=1 >> $O/ab.txt 2>&1
done
echo done
