#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/t2_tc_ab.log; : > $o
timeout 900 python -m pytest tests/test_tc_transforms.py tests/test_stream_transforms.py -q -x 2>&1 | tail -2 >> $o
for i in 1 2; do for e in "STL_T2_TC=1" "STL_T2_TC=0"; do env $e timeout 300 python scripts/t2_tc_ab.py >> $o 2>&1; done; done
cat $o
