#!/bin/bash
o=gpurun_out/noc_split.log; : > $o
for e in STL_STREAM_NOCOMPUTE=0 STL_STREAM_NOCOMPUTE=2 STL_STREAM_NOCOMPUTE=8 STL_STREAM_NOCOMPUTE=10 STL_STREAM_NOCOMPUTE=0; do
  echo "$e $(env $e timeout 300 python scripts/stream_tune.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["enc_us"], d["dec_us"], d["fwd_us"])')" >> $o
done
cat $o
