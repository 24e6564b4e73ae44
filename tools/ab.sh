#!/bin/bash
# A/B timing on the GPU box: bench.py under several settings, alternating, REPS
# times; then (TESTS=1) the GPU tests on the current build.
#   VARIANTS='prev=HF_LIB=paper_2203_08395_b200/libhf_prev.so|cur=|noprefill=HF_PREFILL=0'
set -u
REPS=${REPS:-2}
VARIANTS=${VARIANTS:-"prev=HF_LIB=$PWD/paper_2203_08395_b200/libhf_prev.so|cur="}
mkdir -p gpurun_out/ab
: > gpurun_out/ab/bench.txt
IFS='|' read -ra VS <<< "$VARIANTS"
for r in $(seq $REPS); do for v in "${VS[@]}"; do
  name=${v%%=*}; envs=${v#*=}
  echo "== $name" >> gpurun_out/ab/bench.txt
  env $envs timeout 300 python bench.py ${BENCH_ARGS:-} >> gpurun_out/ab/bench.txt 2>&1
done; done
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest.txt 2>&1
  tail -3 gpurun_out/ab/pytest.txt
fi
