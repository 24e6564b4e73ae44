set -u
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.txt 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/c4.json 2>$O/c4.err
timeout 300 python tools/prop_sweep.py --S 1,4,8,16,32,64 > $O/sweep_C3.txt 2>&1
HF_CONCURRENT=1 timeout 300 python tools/prop_sweep.py --S 1,4,8,16,32,64 > $O/sweep_C3_conc.txt 2>&1
echo done
