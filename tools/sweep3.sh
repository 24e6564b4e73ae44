set -u
OUT=gpurun_out/s3; mkdir -p $OUT/tr
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
HF_TRACE=$OUT/tr/c3 timeout -s KILL 100 python tools/prop_sweep.py --S 1,64 --reps 0 > /dev/null 2>&1
python tools/trace_report.py $OUT/tr/c3_fwd_S1.bin $OUT/tr/c3_bwd_S1.bin $OUT/tr/c3_fwd_S64.bin $OUT/tr/c3_bwd_S64.bin
rm -f $OUT/tr/*.bin
timeout -s KILL 200 python tools/prop_sweep.py --config C5 --S 1,4 --reps 2 2>&1 | tail -3
timeout -s KILL 300 python tools/prop_sweep.py --S 1,4,16,64,256,1024 --reps 3 2>&1 | tail -7
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 -o $OUT/flow python tools/prop_sweep.py --S 64 --once > $OUT/ncu.log 2>&1
