set -u
OUT=gpurun_out/s1; mkdir -p $OUT/tr
P="timeout -s KILL 120 python tools/prop_sweep.py --reps 3"
for cfg in "HF_TW=8 HF_SPLIT=8" "HF_TW=16 HF_SPLIT=8" "HF_TW=16 HF_SPLIT=16" "HF_TW=4 HF_SPLIT=8" "HF_TW=8 HF_SPLIT=8 HF_SLEEP_MAX=64" "HF_TW=8 HF_SPLIT=8 HF_SLEEP_MAX=1024" "HF_SC=32" "HF_SC=16" "HF_CTAS_PER_SM=3"; do
  echo "== $cfg"; env $cfg $P --S 64 2>&1 | tail -1
done
for cfg in "HF_TW=32 HF_SPLIT=16" "HF_TW=16 HF_SPLIT=16" "HF_TW=48 HF_SPLIT=16" "HF_TW=32 HF_SPLIT=8"; do
  echo "== S1 $cfg"; env $cfg $P --S 1 2>&1 | tail -1
done
HF_TRACE=$OUT/tr/c3 timeout -s KILL 100 python tools/prop_sweep.py --S 1,64 --reps 0 > /dev/null 2>&1
python tools/trace_report.py $OUT/tr/c3_fwd_S1.bin $OUT/tr/c3_bwd_S1.bin $OUT/tr/c3_fwd_S64.bin $OUT/tr/c3_bwd_S64.bin
rm -f $OUT/tr/*.bin
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 -o $OUT/flow python tools/prop_sweep.py --S 64 --once > $OUT/ncu.log 2>&1
ls -la $OUT
