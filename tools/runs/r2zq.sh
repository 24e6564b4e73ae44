set -u
# backward with the bitmask poll loop (HF_BWD_MASK=1 build) x backward back-off cap
O=gpurun_out/r2zq; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for rep in 1 2; do
echo "== head" >> $O/ab.txt
timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_SLEEP_MAX_B=96 >> $O/ab.txt 2>&1
echo "== bwd bitmask" >> $O/ab.txt
HF_LIB=$L/libhf_bm.so timeout 600 python tools/env_ab.py --config C4 --S 64 --reps 7 --var "" --var HF_SLEEP_MAX_B=96 --var HF_SLEEP_MAX_B=128 --var HF_SLEEP_MAX_B=192 >> $O/ab.txt 2>&1
done
echo done
