set -u
O=gpurun_out/r2r; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.txt 2>&1
for i in 1 2; do timeout 400 python bench.py > $O/C4_$i.json 2> $O/C4_$i.err; done
timeout 400 python bench.py --config C3 > $O/C3.json 2> $O/C3.err
echo done
