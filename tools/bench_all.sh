#!/bin/bash
# One GPU: a bench line per config (C4 default + C1, C2-*, C3, C5) into $1/
OUT=${1:-gpurun_out/bench}
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/C4.json 2> $OUT/C4.err
for c in C1 C3 C5 C2-chain C2-tree C2-random; do
  python bench.py --config $c --steps 20 --warmup 5 > $OUT/$c.json 2> $OUT/$c.err
done
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/C4.ref.json 2> $OUT/C4.ref.err
