#!/bin/bash
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for T in 0 256 512; do echo "T=$T"; STL_STREAM_T=$T python scripts/transform_probe.py 2>&1 | tail -1; done
STL_STREAM_DEBUG=1 python scripts/transform_probe.py 2>&1 | tail -5
} > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
