set -u
O=gpurun_out/r2z4; mkdir -p $O
timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 2 --var "" > $O/ab1.txt 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary > $O/bench.json 2> $O/bench.err
timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 2 --var "" --var HF_TW=8 > $O/ab2.txt 2>&1
nvidia-smi > $O/smi.txt
echo done
