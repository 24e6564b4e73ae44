set -u
O=gpurun_out/r2x; mkdir -p $O
for S in 64 8; do
for v in "" fakedelay; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-base} S=$S" >> $O/ab.txt
  HF_LIB=$lib timeout 200 python tools/env_ab.py --config C4 --S $S --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
