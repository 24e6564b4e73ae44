set -u
O=gpurun_out/r2zz6; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "batch_small or long_rows" > $O/pytest.txt 2>&1
echo done
