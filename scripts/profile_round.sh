#!/bin/bash
# usage (GPU box): scripts/profile_round.sh <tag>  -> gpurun_out/<tag>_*: bench line, ncu launch list of a short
# bench, ncu --set full of k_score6 / k_replay / k_replay_long / k_mlp / k_mlp_f32 / k_onesweep / k_ff_excursion
T=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py > gpurun_out/${T}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-config5 --no-config4 > /dev/null 2>&1
F="ncu --set full --clock-control none --import-source on"
timeout 600 $F -k regex:k_score6 -s 2 -c 1 -o gpurun_out/${T}_k_score python scripts/prof_score.py 1 > /dev/null 2>&1
timeout 600 $F -k regex:k_replay\$ -c 1 -o gpurun_out/${T}_k_replay python scripts/prof_replay.py 1 > /dev/null 2>&1
timeout 600 $F -k regex:k_replay_long -c 1 -o gpurun_out/${T}_k_replay_long python scripts/prof_replay_long.py 1 > /dev/null 2>&1
timeout 600 $F -k regex:k_mlp\$ -c 1 -o gpurun_out/${T}_k_mlp python scripts/prof_mlp.py 1 bf16 > /dev/null 2>&1
timeout 600 $F -k regex:k_mlp_f32 -c 1 -o gpurun_out/${T}_k_mlp_f32 python scripts/prof_mlp.py 1 fp32 > /dev/null 2>&1
timeout 600 $F -k regex:k_onesweep -s 15 -c 1 -o gpurun_out/${T}_k_onesweep python scripts/prof_sched.py 2 > /dev/null 2>&1
timeout 600 $F -k regex:k_ff_excursion -s 1 -c 1 -o gpurun_out/${T}_k_ff_excursion python scripts/prof_sched.py 2 > /dev/null 2>&1
python scripts/prof_replay_long.py 3 > gpurun_out/${T}_replay_long.log 2>&1
ls -la gpurun_out/ | grep $T
