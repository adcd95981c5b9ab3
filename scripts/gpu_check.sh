#!/bin/bash
# One GPU iteration: parity tests, smoke, short bench. Logs land in gpurun_out/.
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
echo "=== gemm tests"
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "slice_gemm" -p no:cacheprovider 2>&1 | tail -30
echo "=== all gpu tests"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -60
echo "=== smoke"
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
echo "=== bench"
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -20
} > gpurun_out/check.log 2>&1
tail -120 gpurun_out/check.log
