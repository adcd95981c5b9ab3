#!/bin/bash
mkdir -p gpurun_out
{
python scripts/fused_probe.py
STL_FUSED_PAIRS=72 python scripts/fused_probe.py
R=16 STL_FUSED_PAIRS=64 python scripts/fused_probe.py
STL_FUSED_PAIRS=72 timeout 600 ncu --set full --import-source on --clock-control none -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/fused python scripts/fused_probe.py
} > gpurun_out/fused_probe.log 2>&1
grep -v "^==" gpurun_out/fused_probe.log
