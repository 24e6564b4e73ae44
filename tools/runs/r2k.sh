set -u
O=gpurun_out/r2k; mkdir -p $O/tr
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 600 > $O/pytest_wide.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "config_single_full or early_mode_single" > $O/pytest_full.txt 2>&1
timeout 600 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE2=0 --var HF_WIDE2=1 > $O/ab_c5.txt 2>&1
HF_TRACE=$O/tr/c5 timeout 300 python tools/env_ab.py --config C5 --single --reps 1 > $O/run.txt 2>&1
python tools/wide_trace.py $O/tr/c5_w2_fwd.bin $O/tr/c5_w2_bwd.bin > $O/wide2_trace.txt 2>&1
rm -f $O/tr/*.bin
timeout 600 python tools/strong_table.py > $O/strong.txt 2>&1
echo done
