#!/bin/bash
# build experiment copies of libipdg (one per flag set, in parallel) into gpurun_out/ for tools/exp_timing.py
cd "$(dirname "$0")/.."
NCCL=$(python -c "from paper_1801_00246_b200 import build as B; i, l = B.nccl_flags(); print(' '.join(i + l))")
for fs in "$@"; do
  name=$(echo $fs | sed 's/-D//g; s/ /_/g'); [ -z "$name" ] && name=base
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Iinclude $fs paper_1801_00246_b200/csrc/ipdg.cu paper_1801_00246_b200/csrc/refops.cpp -o exp_so/libipdg_exp_$name.so $NCCL 2>/dev/null &
done
wait
