set -u
O=gpurun_out/r2w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 300 > $O/pytest_wide.txt 2>&1
for rep in 1 2; do
for v in "" u2 u8; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-u4}" >> $O/ab.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C5 --single --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --config C5 --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py $O/launches_C5.csv > $O/launches_C5_summary.txt 2>&1
echo done
