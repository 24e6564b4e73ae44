set -u
O=gpurun_out/r2u; mkdir -p $O
HF_WATCHDOG_SPINS=100000 timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 300 > $O/pytest_wide.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "config_single_full or early_mode_single" > $O/pytest_full.txt 2>&1
timeout 600 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE3=0 --var HF_WIDE3=1 > $O/ab_c5.txt 2>&1
bash tools/runs/r2t.sh
cp gpurun_out/r2t/ab.txt $O/ab_rb.txt
echo done
