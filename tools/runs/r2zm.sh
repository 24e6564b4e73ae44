set -u
O=gpurun_out/r2zm; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in one ""; do
echo "== ${lib:-fwd-mask/bwd-old}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 2 -o $O/flow_C4 \
    python bench.py --ncu --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-secondary > $O/ncu_flow.log 2>&1
echo done
