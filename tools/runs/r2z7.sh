set -u
O=gpurun_out/r2z7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invalid.py -m gpu -q -x --timeout 300 -k "batch or tiny or critical or early or scratch or invalid or watchdog" > $O/pytest.txt 2>&1
for i in 1 2; do timeout 400 python bench.py > $O/C4_$i.json 2> $O/C4_$i.err; done
timeout 400 python bench.py --scenarios 256 --no-secondary --no-e2e > $O/C4_S256.json 2> $O/C4_S256.err
timeout 600 python tools/strong_table.py > $O/strong.txt 2>&1
echo done
