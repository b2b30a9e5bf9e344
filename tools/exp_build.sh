#!/bin/bash
# build experimental libraries: impl_<DEG>.cu recompiled with extra -D flags, linked with the in-tree objects
# usage: tools/exp_build.sh DEG name1 "flags1" name2 "flags2" ...   -> exp_so/<name>.so
set -e
DEG=$1; shift
SRCS=${SRCS:-impl_$DEG}
ROOT=$(cd $(dirname $0)/.. && pwd)
NCCL=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -I$ROOT/include -I$NCCL/include"
mkdir -p $ROOT/exp_so
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  ( set -e; objs=""
    for src in $SRCS; do
      nvcc $FL $flags -c $ROOT/paper_1801_00246_b200/csrc/$src.cu -o $ROOT/exp_so/${name}_$src.o > $ROOT/exp_so/${name}_$src.ptxas 2>&1
      objs="$objs $ROOT/exp_so/${name}_$src.o"
    done
    for o in $ROOT/build/obj/*.o; do
      b=$(basename $o .o); case " $SRCS " in *" $b "*) ;; *) objs="$objs $o";; esac
    done
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs -o $ROOT/exp_so/$name.so \
      -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib && echo "built $name" ) &
done
wait
