set -u
O=gpurun_out/r2y; mkdir -p $O
HF_WATCHDOG_SPINS=100000 timeout 600 python -m pytest tests/test_gpu_wide.py -m gpu -q -x --timeout 120 > $O/pytest_wide.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 200 -k "config_single_full or early_mode_single" > $O/pytest_full.txt 2>&1
timeout 600 python tools/env_ab.py --config C5 --single --reps 5 --var HF_WIDE4=0 --var HF_WIDE4=1 > $O/ab_c5.txt 2>&1
echo done
