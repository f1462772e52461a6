#!/bin/bash
# Build the C-ABI library of git revision $1 into build_ab/$2/libmoe_sm100.so (same-box A/B timing:
# run bench.py / scripts/gemm_breakdown.py with MOE_LIB=build_ab/$2/libmoe_sm100.so).
set -e
# REV = WORKTREE copies the working tree; $3 = extra nvcc flags (e.g. -DMOE_EXPERIMENTS).
REV=$1; NAME=$2; EXTRA=$3; D=build_ab/$NAME
rm -rf $D; mkdir -p $D/src $D/include
if [ "$REV" = WORKTREE ]; then
  cp paper_2501_16103_b200/csrc/* $D/src/; cp include/*.h $D/include/
else
  for f in $(git ls-tree --name-only $REV paper_2501_16103_b200/csrc/); do git show $REV:$f > $D/src/$(basename $f); done
  for f in $(git ls-tree --name-only $REV include/); do git show $REV:$f > $D/include/$(basename $f); done
fi
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I $D/include -I $D/src --expt-relaxed-constexpr $EXTRA"
OBJS=""
for f in $D/src/*.cu; do $NV -c $f -o $f.o; OBJS="$OBJS $f.o"; done
for f in $D/src/*.cpp; do g++ -O2 -std=c++17 -fPIC -I $D/include -I $D/src -I /usr/local/cuda/include -c $f -o $f.o; OBJS="$OBJS $f.o"; done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o $D/libmoe_sm100.so $OBJS -lrt -ldl -lpthread
echo $D/libmoe_sm100.so
