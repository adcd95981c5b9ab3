#!/bin/bash
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
python scripts/transform_probe.py 2>&1 | tail -1
STL_STREAM_DEBUG=1 python scripts/transform_probe.py 2>&1 | tail -5 | head -4
timeout 300 python bench.py --steps 50 --warmup 5 --no-extras --no-cpu-baseline | cut -c150-300
} > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
