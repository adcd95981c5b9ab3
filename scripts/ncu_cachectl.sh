#!/bin/bash
# config-2 step kernels under ncu with and without the L2 flush between kernels: does the L2
# state left by the previous kernel (dirty lines) explain the in-pipeline slowdown?
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control all -k regex:"k_stream|slice_gemm" -s 10 -c 10 --csv --log-file gpurun_out/cc_all.csv $B > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:"k_stream|slice_gemm" -s 10 -c 10 --csv --log-file gpurun_out/cc_none.csv $B > /dev/null 2>&1
ls -la gpurun_out/cc_*.csv
