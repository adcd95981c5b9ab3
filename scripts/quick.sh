#!/bin/bash
# tests + transform probe + short bench
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 300 python scripts/transform_probe.py
timeout 300 python scripts/fused_probe.py 2>&1 | grep '"fused": 0'
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -3
} > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
