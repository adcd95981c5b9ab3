#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/order1_ab.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
STL_LIB=$P STL_GEMM_ORDER1=0 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "8192 or full" 2>&1 | tail -1 >> $o
for i in 1 2 3; do for e in "STL_GEMM_ORDER1=-1" "STL_GEMM_ORDER1=0" "STL_GEMM_ORDER1=2"; do
  echo "$e $(env STL_LIB=$P $e timeout 300 python scripts/north_star.py 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["burst"]["stl_ms"],4), round(d["burst"]["cublas_ms"],4), round(d["burst"]["speedup"],3))')" >> $o
done; done
bash scripts/ab_step.sh order1_step "STL_GEMM_ORDER1=-1" "STL_GEMM_ORDER1=0" 2
cat gpurun_out/order1_step.log >> $o
cat $o
