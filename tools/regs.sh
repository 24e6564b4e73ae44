#!/bin/bash
# register / spill summary of the kernels in one .cu file:
#   tools/regs.sh file.cu [regex] [extra nvcc flags...]
f=$1; pat=${2:-.}; shift; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr -ftz=false -I include "$@" -c $f -o /tmp/regs_$$.o 2>&1 | \
  awk '/Compiling entry function/ {match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, RLENGTH); sp="0"}
       /bytes spill stores/ {match($0, /[0-9]+ bytes spill stores/); sp=substr($0, RSTART, RLENGTH-18)}
       /Used [0-9]+ registers/ {match($0, /Used [0-9]+ registers/); r=substr($0, RSTART+5, RLENGTH-15);
         print r "\tspill=" sp "\t" name}' | c++filt | grep -E "$pat" | sed 's/hf::(anonymous namespace):://g; s/(FlowParams)//'
rm -f /tmp/regs_$$.o
