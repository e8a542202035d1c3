#!/bin/bash
# build libmt.so from the csrc of a git revision (or the working tree with REV=WT) into OUT
# usage: REV=<rev|WT> OUT=ab/A.so bash tools/build_variant.sh
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
if [ "$REV" = "WT" ]; then mkdir -p $TMP/paper_2111_14255_b200; cp -r $ROOT/paper_2111_14255_b200/csrc $TMP/paper_2111_14255_b200/; cp -r $ROOT/include $TMP/
else git -C $ROOT archive $REV paper_2111_14255_b200/csrc include | tar -x -C $TMP; fi
S=$TMP/paper_2111_14255_b200/csrc
mkdir -p $(dirname $ROOT/$OUT)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared \
  --expt-relaxed-constexpr $NVFLAGS -o $ROOT/$OUT $S/kernels.cu $S/kernels_cr.cu $S/host.cpp $S/plan.cpp -ldl -lpthread -lrt
rm -rf $TMP
