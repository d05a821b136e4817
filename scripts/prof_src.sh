#!/bin/bash
# usage: scripts/prof_src.sh <tag>  (on the GPU box) -> gpurun_out/<tag>.ncu-rep (ncu --set full of one k_score4 launch)
ncu --set full --clock-control none --import-source on -k regex:k_score4 -s 2 -c 1 -o gpurun_out/$1 python scripts/prof_score.py 1 > gpurun_out/$1.log 2>&1
tail -1 gpurun_out/$1.log
