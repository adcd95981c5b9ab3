#!/bin/bash
mkdir -p gpurun_out
for sel in "t2 and 64-2048-24" "encode_decode_bf16 and 24-36-256" "encode_decode_bf16 and 24-64-2304"; do
  echo "== $sel"
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 --target-processes all \
    python -m pytest tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider -k "$sel" 2>&1 | grep -vE "^\.+|passed" | grep -E "RACECHECK SUMMARY|Race reported|in k_|at |__global__|kernel|Write|Read|smem|shared" | head -24
done
