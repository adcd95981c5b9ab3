#!/bin/bash
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -1
o=gpurun_out/tail_ab.log; : > $o
for i in 1 2; do for e in STL_STREAM_TAIL=2 STL_STREAM_TAIL=0 STL_STREAM_TAIL=4; do
  echo "$e $(env $e timeout 300 python scripts/stream_tune.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["enc_us"], d["dec_us"], d["fwd_us"], d["h"])')" >> $o
done; done
cat $o
STL_STREAM_TAIL=2 python scripts/trace_fwd.py 2>&1 | tail -4
bash scripts/ab_step.sh ab_tail "STL_STREAM_TAIL=2" "STL_STREAM_TAIL=0" 2
