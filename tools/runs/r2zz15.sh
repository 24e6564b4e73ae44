set -u
# gathers in flight per lane (RB4_FWD / RB4_BWD) with the final kernels
O=gpurun_out/r2zz15; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in "" rbf3 rbf5 rbb3; do
echo "== ${lib:-head (RB 4/4)}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
HF_LIB=$L/libhf_rbf3.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var HF_TW_F=8 --var HF_TW_F=9 --var HF_TW_F=10 >> $O/ab.txt 2>&1
echo done
