set -u
O=gpurun_out/r2d; mkdir -p $O/tr
for S in 64 8 1; do
timeout 600 python tools/env_ab.py --config C4 --S $S --reps 5 --var HF_PRED_PCT=0 --var HF_PRED_PCT=50 --var HF_PRED_PCT=70 --var HF_PRED_PCT=85 --var HF_PRED_PCT=70,HF_PRED_MIN=1000 > $O/ab_S$S.txt 2>&1
done
HF_TRACE=$O/tr/c3 timeout 200 python tools/prop_sweep.py --S 8,64 --reps 0 > $O/trace_run.txt 2>&1
python tools/trace_report.py $O/tr/c3_fwd_S8.bin $O/tr/c3_bwd_S8.bin $O/tr/c3_fwd_S64.bin $O/tr/c3_bwd_S64.bin > $O/trace_C3.txt 2>&1
rm -f $O/tr/*.bin
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "batch or tiny or full_c3" > $O/pytest.txt 2>&1
echo done
