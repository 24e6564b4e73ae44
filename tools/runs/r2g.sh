set -u
O=gpurun_out/r2g; mkdir -p $O/tr
HF_TRACE=$O/tr/c5 timeout 300 python tools/env_ab.py --config C5 --single --reps 1 > $O/run.txt 2>&1
python tools/wide_trace.py $O/tr/c5_w1_fwd.bin $O/tr/c5_w1_bwd.bin > $O/wide_trace.txt 2>&1
rm -f $O/tr/*.bin
echo done
