#!/bin/bash
# ncu --set full on the transform kernels of one config-2 layer step (+ launch list)
tag=${1:-r01b}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_encode|k_decode|k_tiles|k_planes" -s 8 -c 4 -o gpurun_out/${tag}_xf $B > gpurun_out/${tag}_xf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc2_kernel" -s 6 -c 3 -o gpurun_out/${tag}_gemm $B > gpurun_out/${tag}_gemm.log 2>&1
ls gpurun_out
