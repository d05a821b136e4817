#!/bin/bash
# usage (GPU box): scripts/ab_replay.sh v1 v2 ...  -> replay time per library build ab_variants/<v>.so, interleaved x3
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; RTLM_LIB=ab_variants/$v.so python scripts/prof_replay.py 10 2>&1 | tail -1
  done
done
