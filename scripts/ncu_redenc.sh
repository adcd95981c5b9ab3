#!/bin/bash
# ncu of the encode + g_d reduction: tcgen05 variant (probe STL_RED_TC=1, 256- and 512-tile
# units) next to the mma.sync k_stream<kEncRed>
mkdir -p gpurun_out
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --no-t2t --no-sweep"
STL_LIB=$P STL_RED_TC=1 timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_red_tc<.bool.1" -s 2 -c 1 -o gpurun_out/ncu_redenc256 $B > gpurun_out/ncu_redenc.log 2>&1
STL_LIB=$P STL_RED_TC=1 STL_RED_TC_T=512 timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_red_tc<.bool.1" -s 2 -c 1 -o gpurun_out/ncu_redenc512 $B >> gpurun_out/ncu_redenc.log 2>&1
STL_LIB=$P timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_stream<.int.1," -s 2 -c 1 -o gpurun_out/ncu_encred_mma $B >> gpurun_out/ncu_redenc.log 2>&1
ls -la gpurun_out/*.ncu-rep
