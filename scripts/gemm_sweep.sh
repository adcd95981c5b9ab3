#!/bin/bash
mkdir -p gpurun_out
{ python scripts/gemm_bench.py; STL_GEMM_L2PF=1 python scripts/gemm_bench.py; STL_GEMM_L2PF=1 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k gemm 2>&1 | tail -2; } > gpurun_out/gemm_sweep.log 2>&1
cat gpurun_out/gemm_sweep.log
