#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/groups_ab.log; : > $o
run() { env "$@" timeout 300 python scripts/stream_tune.py >> $o 2>&1; }
run STL_X=base
run STL_STREAM_GROUPS=4
run STL_STREAM_GROUPS=4 STL_STREAM_T=512
run STL_STREAM_GROUPS=4 STL_STREAM_NBUF=2
run STL_STREAM_GROUPS=4 STL_STREAM_NBUF=3
cat $o
bash scripts/ab_step.sh ab_groups "STL_X=base" "STL_STREAM_GROUPS=4" 2
