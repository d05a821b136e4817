#!/bin/bash
# usage (GPU box): scripts/profile_round.sh <tag>  -> gpurun_out/<tag>_*: bench line, config-4 line,
# ncu launch list of a short bench, ncu --set full of k_score4 / k_replay / k_mlp
T=$1
python bench.py > gpurun_out/${T}_bench.log 2>&1
python bench.py --no-cpu-baseline --no-mlp --no-traces --no-config5 --steps 3 > gpurun_out/${T}_config4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score4 -s 2 -c 1 -o gpurun_out/${T}_k_score python scripts/prof_score.py 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -c 1 -o gpurun_out/${T}_k_replay python scripts/prof_replay.py 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp -c 1 -o gpurun_out/${T}_k_mlp python scripts/prof_mlp.py 1 > /dev/null 2>&1
ls -la gpurun_out/ | grep $T
