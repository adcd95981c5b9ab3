#!/bin/bash
# racecheck (full report) on the tcgen05 kernels, parity tests, then the reductions' dynamic
# tail A/B on the config-2 step (and the tcgen05 encode-reduction with it)
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 12 --target-processes all \
  python -m pytest tests/test_tc_transforms.py -m gpu -q -x -p no:cacheprovider \
  -k "(tc_encode_decode and 24-12-2304) or (tc_decode_reduction and 24) or (tc_remix_chain and 24)" \
  > gpurun_out/racecheck_tc.log 2>&1
o=gpurun_out/reddyn_ab.log; : > $o
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_tc_transforms.py -q -x 2>&1 | tail -2 >> $o
bash scripts/ab_step.sh reddyn_step "STL_RED_DYN=1" "STL_RED_DYN=0" 3
cat gpurun_out/reddyn_step.log >> $o
bash scripts/ab_step.sh reddyn_enc "STL_RED_TC=1 STL_RED_TC_T=512" "STL_RED_TC=1" 2
cat gpurun_out/reddyn_enc.log >> $o
cat $o
