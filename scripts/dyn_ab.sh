#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -1
o=gpurun_out/dyn_ab.log; : > $o
for i in 1 2; do
for e in STL_STREAM_DYNAMIC=1 STL_STREAM_DYNAMIC=0; do env $e timeout 300 python scripts/stream_tune.py >> $o 2>&1; done
done
cat $o | cut -c1-250
STL_STREAM_DYNAMIC=1 python scripts/trace_fwd.py 2>&1 | tail -4
bash scripts/ab_step.sh ab_dyn "STL_STREAM_DYNAMIC=1" "STL_STREAM_DYNAMIC=0" 2
