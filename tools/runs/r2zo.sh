set -u
# backward registers: partials in flight (PW_BWD) x minimum blocks per SM (6 / 7)
O=gpurun_out/r2zo; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
for lib in "" b6p2 b7p2 b7p1 b6p1; do
echo "== ${lib:-head (PW 4, 96 regs)}" >> $O/ab.txt
HF_LIB=$L/libhf${lib:+_$lib}.so timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" >> $O/ab.txt 2>&1
done; done
echo done
