#!/bin/bash
mkdir -p gpurun_out
tag=${1:-gemm}
ITERS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 3 -c 1 -o gpurun_out/${tag} python scripts/gemm_bench.py cfg2_fwd > gpurun_out/${tag}.log 2>&1
ls -la gpurun_out | grep ${tag}
