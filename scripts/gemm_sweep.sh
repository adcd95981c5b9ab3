#!/bin/bash
mkdir -p gpurun_out
{ STL_GEMM_MC=1 timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or layer or batched or f24" 2>&1 | tail -2
for mc in 0 1 0 1; do echo "mc=$mc"; STL_GEMM_MC=$mc python scripts/gemm_bench.py | cut -c1-100; STL_GEMM_MC=$mc python scripts/transform_probe.py | tail -1 | cut -c1-250; done
} > gpurun_out/gemm_sweep.log 2>&1
cat gpurun_out/gemm_sweep.log
