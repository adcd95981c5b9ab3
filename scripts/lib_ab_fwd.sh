#!/bin/bash
# A/B of two library builds on the forward (config 2 and 8192^3) and the config-2 step
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
  echo old; STL_LIB=$PWD/scripts/ab/lib_old.so timeout 300 python scripts/fused_probe.py 2>&1 | grep '"fused": 0' | cut -c1-200
  STL_LIB=$PWD/scripts/ab/lib_old.so timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-200
  echo new; timeout 300 python scripts/fused_probe.py 2>&1 | grep '"fused": 0' | cut -c1-200
  timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-200
done
} > gpurun_out/lib_ab_fwd.log 2>&1
cat gpurun_out/lib_ab_fwd.log
