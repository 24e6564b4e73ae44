set -u
# backward bitmask poll loop: free registers (125) vs 5 blocks/SM (96)
O=gpurun_out/r2zz7; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in "" bm bm5; do
echo "== ${lib:-head}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 256 --reps 3 --var "" >> $O/ab.txt 2>&1
done; done
echo done
