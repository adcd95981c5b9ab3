#!/bin/bash
mkdir -p gpurun_out
{
for o in 0 1; do for pr in 0 1; do echo "pdl=$o profile=$pr"; STL_BENCH_PROFILE=$pr STL_PDL=$o timeout 300 python bench.py --steps 50 --warmup 5 --no-extras --no-cpu-baseline | cut -c150-300; done; done
} > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
