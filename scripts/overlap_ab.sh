#!/bin/bash
# GEMM -> decode overlap of the cache-less forward (STL_FWD_OVERLAP, probe library): parity
# tests and stress with it on, then the north-star comparison on vs off (alternating runs)
mkdir -p gpurun_out
o=gpurun_out/overlap_ab.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
STL_LIB=$P STL_FWD_OVERLAP=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_tc_transforms.py tests/test_stream_transforms.py -q -x 2>&1 | tail -2 >> $o
STL_LIB=$P STL_FWD_OVERLAP=1 FWDS=400 STEPS=50 CHAINS=20 timeout 600 python scripts/stress_tc.py 2>&1 | tail -4 >> $o
for i in 1 2 3; do for e in "STL_FWD_OVERLAP=1" "STL_FWD_OVERLAP=0"; do
  echo "$e $(env STL_LIB=$P $e timeout 300 python scripts/north_star.py 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["burst"]["stl_ms"],4), round(d["burst"]["cublas_ms"],4), round(d["burst"]["speedup"],3), round(d["sustained"]["speedup"],3))')" >> $o
done; done
cat $o
