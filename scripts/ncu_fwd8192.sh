#!/bin/bash
# ncu --set full (with source) on the 8192^3 forward's encode / decode / slice GEMM
tag=${1:-fwd8192}
mkdir -p gpurun_out
export ITERS=3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_(en|de)code_tc" -s 2 -c 2 \
  -o gpurun_out/${tag}_stream python scripts/fwd8192.py > gpurun_out/${tag}_stream.log 2>&1
ls -la gpurun_out/
