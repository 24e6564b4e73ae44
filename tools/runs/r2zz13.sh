set -u
# long-row cut (LO_SPLIT) and part size (LO_PE) re-checked with the final kernels
O=gpurun_out/r2zz13; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in "" pe16 pe24 sp10 sp6; do
echo "== ${lib:-head (split 8, pe 20)}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
echo done
