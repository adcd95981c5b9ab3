#!/bin/bash
mkdir -p gpurun_out
{
for o in 0 1 2; do echo "overlap=$o"; STL_OVERLAP=$o python scripts/transform_probe.py 2>&1 | tail -1; done
} > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
