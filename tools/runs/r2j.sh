set -u
O=gpurun_out/r2j; mkdir -p $O/tr
for v in "" tw8192 tw4096; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-default16384}" >> $O/ab.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE2=0 --var HF_WIDE2=1 >> $O/ab.txt 2>&1
done
HF_LIB=$PWD/paper_2203_08395_b200/libhf_tw4096.so HF_TRACE=$O/tr/c5 timeout 300 python tools/env_ab.py --config C5 --single --reps 1 > $O/run.txt 2>&1
python tools/wide_trace.py $O/tr/c5_w2_fwd.bin > $O/trace4096.txt 2>&1
rm -f $O/tr/*.bin
echo done
