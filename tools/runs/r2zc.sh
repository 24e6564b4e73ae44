set -u
# re-entry check of the current tree + globaltimer resolution
O=gpurun_out/r2zc; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $O/gpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/timer_res tools/dbg/timer_res.cu && /tmp/timer_res > $O/timer_res.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.txt 2>&1
timeout 400 python bench.py > $O/C4.json 2> $O/C4.err
timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" > $O/ab.txt 2>&1
echo done
