#!/bin/bash
# A/B of probe switches on the config-2 step (bench.py, probe library): alternating runs
# usage: scripts/ab_step.sh <tag> "<envA>" "<envB>" [reps]
mkdir -p gpurun_out
o=gpurun_out/$1.log; : > $o
for i in $(seq ${4:-3}); do
  for e in "$2" "$3"; do
    env STL_LIB=$PWD/paper_2503_12211_b200/libstl_b200_probe.so $e timeout 300 python bench.py --steps 50 --warmup 10 --no-extras --no-cpu-baseline --no-t2t --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})" >> $o
  done
done
cat $o
