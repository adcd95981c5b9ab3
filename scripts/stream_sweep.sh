#!/bin/bash
mkdir -p gpurun_out
for cfg in "0 0" "256 0" "512 0" "0 1"; do
  set -- $cfg
  echo "T=$1 nocompute=$2"
  STL_STREAM_T=$1 STL_STREAM_NOCOMPUTE=$2 python scripts/transform_probe.py 2>&1 | head -1
done > gpurun_out/sweep.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 >> gpurun_out/sweep.log
cat gpurun_out/sweep.log
