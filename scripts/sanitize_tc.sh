#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the tcgen05 transforms (K10-K13)
mkdir -p gpurun_out
SEL='(tc_encode_decode and (12-2304 and (24 or 9 or 32))) or (tc_decode_reduction and 24) or (tc_remix_chain and 24)'
{
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard --print-limit 8"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_tc_transforms.py -m gpu -q -x -p no:cacheprovider -k "$SEL" 2>&1 | grep -vE "^\.+ *\[" | tail -12
  echo "rc=${PIPESTATUS[0]}"
done
} > gpurun_out/sanitize_tc.log 2>&1
cat gpurun_out/sanitize_tc.log
