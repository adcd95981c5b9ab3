#!/bin/bash
mkdir -p gpurun_out
{
python scripts/gemm_bench.py
STL_GEMM_1CTA=1 python scripts/gemm_bench.py
ITERS=3 timeout 600 ncu --set full --clock-control none -k regex:tc2_kernel -s 5 -c 1 -o gpurun_out/g2 python scripts/gemm_bench.py cfg2_fwd
} > gpurun_out/gemm_probe.log 2>&1
cat gpurun_out/gemm_probe.log | grep -v "^==PROF=="
