#!/bin/bash
# A/B of two library builds on the config-2 step: scripts/ab/lib_old.so vs the in-tree build
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do
  echo old; STL_LIB=$PWD/scripts/ab/lib_old.so timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-260
  echo new; timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-260
done
} > gpurun_out/lib_ab.log 2>&1
cat gpurun_out/lib_ab.log
