#!/bin/bash
# usage: scripts/build_variant.sh <name> [git-rev]  -> ab_variants/<name>.so (librtlm.so built from the working
# tree, or from the csrc/ + include/ of a commit), for scripts/ab_score.sh A/B timing on the GPU box
set -e
N=$1; REV=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $ROOT/ab_variants
if [ -n "$REV" ]; then
  W=$(mktemp -d); mkdir -p $W/paper_2309_06619_b200/csrc $W/include
  git -C $ROOT archive $REV paper_2309_06619_b200/csrc include | tar -x -C $W
  SRC=$W
else
  SRC=$ROOT
fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -o $ROOT/ab_variants/$N.so $SRC/paper_2309_06619_b200/csrc/*.cu $EXTRA_NVCC
echo built ab_variants/$N.so
