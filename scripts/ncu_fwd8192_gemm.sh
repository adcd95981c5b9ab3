#!/bin/bash
# ncu --set full on the 8192^3 forward's slice GEMM (north-star tensor-pipe evidence) and the
# dram bytes of all three launches of one forward
tag=${1:-fwd8192_gemm}
mkdir -p gpurun_out
export ITERS=3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slice_gemm -s 1 -c 1 \
  -o gpurun_out/${tag} python scripts/fwd8192.py > gpurun_out/${tag}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -s 3 -c 3 --csv \
  --log-file gpurun_out/${tag}_fwd_bytes.csv python scripts/fwd8192.py > /dev/null 2>&1
cat gpurun_out/${tag}_fwd_bytes.csv | tail -14
