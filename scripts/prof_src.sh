#!/bin/bash
# usage: scripts/prof_src.sh <tag> [kernel regex, default k_score6]  (on the GPU box)
#   -> gpurun_out/<tag>.ncu-rep (ncu --set full of one scoring launch) + <tag>_src.csv (source page) + <tag>_raw.csv
K=${2:-k_score6}
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/$1 python scripts/prof_score.py 1 > gpurun_out/$1.log 2>&1
tail -1 gpurun_out/$1.log
ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$1_src.csv 2>/dev/null
ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
