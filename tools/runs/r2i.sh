set -u
O=gpurun_out/r2i; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide2 -c 1 -o $O/wide2 python bench.py --config C5 --ncu --steps 1 --warmup 0 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/wide2.ncu-rep > $O/sum.txt 2>&1
python tools/ncu_stalls.py $O/wide2.ncu-rep k_wide2 40 > $O/stalls.txt 2>&1
ncu -i $O/wide2.ncu-rep --page source --csv --print-source cuda > $O/src_cuda.csv 2>&1
for v in "" ef; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-default}" >> $O/ab_ef.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" >> $O/ab_ef.txt 2>&1
done
echo done
