#!/bin/bash
# ncu evidence for one build: launch list of a short bench + full sets of the top kernels.
# usage: scripts/ncu_capture.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slice_gemm_tc \
  -s 6 -c 2 -o gpurun_out/${tag}_gemm $B > gpurun_out/${tag}_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_(en|de)code_tc|k_red_tc" \
  -s 12 -c 6 -o gpurun_out/${tag}_stream $B > gpurun_out/${tag}_stream.log 2>&1
ls -la gpurun_out/
