#!/bin/bash
# A/B of the product library (new) against a saved copy (old) on the 8192^3 forward, interleaved
o=gpurun_out/micro_ab.log; : > $o
for i in 1 2 3; do
  for L in paper_2503_12211_b200/libstl_b200_probe.so build_ab/old_probe.so; do
    echo "$L $(STL_LIB=$PWD/$L timeout 300 python scripts/stream_tune.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["enc_us"], d["dec_us"], d["fwd_us"])')" >> $o
  done
done
cat $o
