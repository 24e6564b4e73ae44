set -u
O=gpurun_out/r2zl; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in one ""; do
echo "== ${lib:-fwd-mask/bwd-slot}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
