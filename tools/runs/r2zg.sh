set -u
# diagnostic: k_flow with always-final gathers (-DHF_DBG_FAKE_GATHER, wrong results)
O=gpurun_out/r2zg; mkdir -p $O
L=$PWD/paper_2203_08395_b200
for S in 64 8; do
echo "== base S=$S" >> $O/ab.txt
HF_LIB=$L/libhf_base.so timeout 300 python tools/env_ab.py --config C4 --S $S --reps 5 --var "" >> $O/ab.txt 2>&1
echo "== fake gathers S=$S" >> $O/ab.txt
HF_LIB=$L/libhf_fakeg.so timeout 300 python tools/env_ab.py --config C4 --S $S --reps 5 --var "" --var HF_SLEEP_MAX=32 >> $O/ab.txt 2>&1
done
echo done
