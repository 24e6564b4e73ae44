set -u
# validation of the single-chunk kernel + forward poll bitmask: GPU tests, smoke, bench lines
O=gpurun_out/r2zp; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.txt 2>&1
for i in 1 2; do timeout 400 python bench.py > $O/C4_$i.json 2> $O/C4_$i.err; done
for c in C3 C1; do timeout 400 python bench.py --config $c > $O/$c.json 2> $O/$c.err; done
for s in 256 1024; do timeout 900 python bench.py --scenarios $s --no-secondary --no-e2e > $O/C4_S$s.json 2> $O/C4_S$s.err; done
echo done > $O/done.txt
