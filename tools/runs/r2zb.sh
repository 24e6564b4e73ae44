set -u
O=gpurun_out/r2zb; mkdir -p $O
for S in 1 2 4 8 12; do
  timeout 300 python tools/env_ab.py --config C4 --S $S --reps 7 --var HF_CONCURRENT=0 --var HF_CONCURRENT=1 >> $O/ab_conc.txt 2>&1
done
timeout 900 python tools/env_ab.py --config C4 --S 256 --reps 5 --var "" > $O/ab256.txt 2>&1
echo done
