set -u
# fake-gather diagnostic on the final kernels (throughput floor without dependency waits)
O=gpurun_out/r2zz4; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for S in 64 8; do
echo "== final S=$S" >> $O/ab.txt
timeout 300 python tools/env_ab.py --config C4 --S $S --reps 5 --var "" >> $O/ab.txt 2>&1
echo "== fake gathers S=$S" >> $O/ab.txt
HF_LIB=$L/libhf_fakeg.so timeout 300 python tools/env_ab.py --config C4 --S $S --reps 5 --var "" >> $O/ab.txt 2>&1
done
echo done
