#!/bin/bash
# ncu --set full of the tcgen05 encode / decode and the mma.sync streaming ones at 8192^3
mkdir -p gpurun_out
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(en|de)code_tc" -s 2 -c 2 -o gpurun_out/ncu_tc python scripts/tc_one.py > gpurun_out/ncu_tc.log 2>&1
STL_LIB=$P STL_ENC_TC=0 STL_DEC_TC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream" -s 2 -c 2 -o gpurun_out/ncu_mma python scripts/tc_one.py > gpurun_out/ncu_mma.log 2>&1
ls -la gpurun_out/*.ncu-rep
