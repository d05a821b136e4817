#!/bin/bash
# usage (GPU box): scripts/gpu_round.sh <tag> [pytest -k expr]  -> gpurun_out/<tag>_{gputest,bench}.log
T=$1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -x -q $K > gpurun_out/${T}_gputest.log 2>&1
tail -5 gpurun_out/${T}_gputest.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1
tail -c 600 gpurun_out/${T}_bench.log
