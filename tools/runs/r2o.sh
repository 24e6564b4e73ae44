set -u
O=gpurun_out/r2o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kahn_async.py -m gpu -q -x --timeout 600 > $O/pytest_kahn_async.txt 2>&1
for c in C3 C5 C2-random C2-chain C2-tree; do
  for a in 0 1; do
    echo "== $c HF_KAHN_ASYNC=$a" >> $O/lev.txt
    HF_KAHN_ASYNC=$a HF_LEV_TIMES=1 timeout 300 python bench.py --config C2-random --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > /dev/null 2>&1
    HF_KAHN_ASYNC=$a HF_LEV_TIMES=1 timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-secondary --steps 5 --warmup 3 2>&1 | grep "levelize stages" | tail -1 >> $O/lev.txt
  done
done
for v in "" pw8 pw16; do
  lib=""; [ -n "$v" ] && lib=$PWD/paper_2203_08395_b200/libhf_$v.so
  echo "== ${v:-pw4}" >> $O/ab_pw.txt
  HF_LIB=$lib timeout 300 python tools/env_ab.py --config C4 --S 64 --reps 5 --var "" >> $O/ab_pw.txt 2>&1
done
echo done
