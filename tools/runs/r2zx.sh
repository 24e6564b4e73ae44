set -u
O=gpurun_out/r2zx; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q --timeout 600 > $O/pytest.txt 2>&1
echo done
