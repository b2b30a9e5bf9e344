#!/bin/bash
# run a timing script against experimental library builds in exp_so/ (each copied over the in-tree one)
# usage: tools/exp_run.sh "<python args>" [names...]   (default: every exp_so/*.so)
args=$1; shift
names=${@:-$(ls exp_so/*.so | xargs -n1 basename | sed 's/\.so$//')}
cp paper_1801_00246_b200/libipdg.so /tmp/libipdg_intree.so
for n in $names; do
  cp exp_so/$n.so paper_1801_00246_b200/libipdg.so
  touch paper_1801_00246_b200/libipdg.so
  echo "== $n"
  timeout 600 python $args 2>&1 | tail -20
done
cp /tmp/libipdg_intree.so paper_1801_00246_b200/libipdg.so
