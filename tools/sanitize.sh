#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) over the small GPU tests (C1-sized
# and scaled graphs: golden graphs, tiny DAGs, batches incl. S=64, the wide S=1 path,
# critical path / top-K, MIS): shared-memory races and barrier misuse in every kernel
# those tests launch.  Output: gpurun_out/sanitize/<tool>.txt
set -u
O=gpurun_out/sanitize; mkdir -p $O
SEL="golden or tiny or batch_small or long_rows and 64 or isolated or multi_edges or empty or critical_path_integer or top_k_device and 0.004 or mis_ties or early_mode_tiny or config_single and C1"
for tool in racecheck synccheck memcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 2400 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -q -p no:cacheprovider \
    -k "$SEL" > $O/$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
  tail -3 $O/$tool.txt >> $O/summary.txt
done
