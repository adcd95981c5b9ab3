#!/bin/bash
mkdir -p gpurun_out
{ python scripts/gemm_bench.py; STL_GEMM_BN=128 python scripts/gemm_bench.py; python scripts/transform_probe.py | tail -1; STL_GEMM_BN=128 python scripts/transform_probe.py | tail -1; } > gpurun_out/gemm_sweep.log 2>&1
cat gpurun_out/gemm_sweep.log
