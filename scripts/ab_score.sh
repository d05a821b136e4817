#!/bin/bash
# usage (GPU box): scripts/ab_score.sh v1 v2 ...  -> k_score time per library build ab_variants/<v>.so, interleaved x3
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; RTLM_LIB=ab_variants/$v.so python scripts/prof_score.py 20 | sed 's/.*min/min/'
  done
done
