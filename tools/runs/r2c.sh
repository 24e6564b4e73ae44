set -u
O=gpurun_out/r2c; mkdir -p $O/tr
HF_TRACE=$O/tr/c3 timeout 200 python tools/prop_sweep.py --S 1,8,64 --reps 0 > $O/trace_run.txt 2>&1
python tools/trace_report.py $O/tr/c3_fwd_S1.bin $O/tr/c3_bwd_S1.bin $O/tr/c3_fwd_S8.bin $O/tr/c3_bwd_S8.bin $O/tr/c3_fwd_S64.bin $O/tr/c3_bwd_S64.bin > $O/trace_C3.txt 2>&1
rm -f $O/tr/*.bin
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "view_sweep or top_k or full_c4 or critical" > $O/pytest.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wide -c 2 -o $O/wide python bench.py --config C5 --ncu --steps 1 --warmup 0 > $O/ncu_wide.log 2>&1
python tools/ncu_summary.py $O/wide.ncu-rep > $O/ncu_wide_summary.txt 2>&1
python tools/ncu_stalls.py $O/wide.ncu-rep k_wide 20 > $O/ncu_wide_stalls.txt 2>&1
echo done
