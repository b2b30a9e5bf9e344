#!/bin/bash
# run a timing script against every experimental library build in exp_so/ (each copied over the in-tree one)
# usage: tools/exp_run.sh "<python args>"   (output: gpurun_out/exp_<name>.log)
for f in exp_so/*.so; do
  n=$(basename $f .so)
  cp $f paper_1801_00246_b200/libipdg.so
  touch paper_1801_00246_b200/libipdg.so
  echo "== $n"
  timeout 600 python $1 2>&1 | grep -v '^{"N"' | tail -20
done
