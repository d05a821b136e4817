#!/bin/bash
# usage (GPU box): scripts/ab_mlp.sh <precision> v1 v2 ...  -> MLP time per library build ab_variants/<v>.so, x3
P=$1; shift
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; RTLM_LIB=ab_variants/$v.so python scripts/prof_mlp.py 10 $P 2>&1 | tail -1 | sed 's/.*min/min/'
  done
done
