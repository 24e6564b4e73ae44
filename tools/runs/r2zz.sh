set -u
# backward partials in flight per group: 4 (default) / 6 / 8
O=gpurun_out/r2zz; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in "" pw6 pw8; do
echo "== ${lib:-pw4}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 8 --reps 5 --var "" >> $O/ab.txt 2>&1
done; done
echo done
