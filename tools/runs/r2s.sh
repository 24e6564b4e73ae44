set -u
O=gpurun_out/r2s; mkdir -p $O
for b in 1024 512 256 128; do
  echo "== HF_KAHN_BLOCK=$b" >> $O/kahn_block.txt
  HF_KAHN_BLOCK=$b HF_LEV_TIMES=1 timeout 300 python bench.py --config C3 --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 2>&1 | grep "levelize stages" | tail -1 >> $O/kahn_block.txt
done
bash tools/sanitize.sh
cp gpurun_out/sanitize/* $O/ 2>/dev/null
echo done
