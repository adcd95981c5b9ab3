#!/bin/bash
# ncu --set full on the streaming transform kernels of one config-2 layer step
tag=${1:-stream}
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream" -s 4 -c 4 -o gpurun_out/${tag} $B > gpurun_out/${tag}.log 2>&1
ls -la gpurun_out
