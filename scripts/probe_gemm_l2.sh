#!/bin/bash
# L2-boundness probe of the slice GEMM: timings (+ mainloop-only) and ncu of ours vs cuBLAS.
mkdir -p gpurun_out
export STL_LIB=paper_2503_12211_b200/libstl_b200_probe.so  # STL_* switches: probe build
tag=${1:-l2probe}
{
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python scripts/probe_gemm_l2.py all
STL_GEMM_NOSTORE=1 timeout 300 python scripts/probe_gemm_l2.py stl
STL_GEMM_DEBUG=1 ITERS=3 timeout 300 python scripts/probe_gemm_l2.py stl 2>&1 | tail -3
} > gpurun_out/${tag}.log 2>&1
METRICS=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_requests_srcunit_tex.sum,lts__d_sectors.sum,lts__cycles_elapsed.avg.per_second
ITERS=2 timeout 600 ncu --metrics $METRICS --clock-control none -k regex:tc2_kernel -s 2 -c 1 --csv python scripts/probe_gemm_l2.py stl > gpurun_out/${tag}_ncu_stl.csv 2>&1
ITERS=2 timeout 600 ncu --metrics $METRICS --clock-control none -k regex:"nvjet|gemm|cutlass|sm100" -s 3 -c 1 --csv python scripts/probe_gemm_l2.py bmm > gpurun_out/${tag}_ncu_bmm.csv 2>&1
ITERS=2 timeout 600 ncu --metrics $METRICS --clock-control none -k regex:"nvjet|gemm|cutlass|sm100" -s 3 -c 1 --csv python scripts/probe_gemm_l2.py dense > gpurun_out/${tag}_ncu_dense.csv 2>&1
cat gpurun_out/${tag}.log
