#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/overlap_ab2.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for i in 1 2 3; do for e in "STL_FWD_OVERLAP=1 STL_TC_DYN=-1" "STL_FWD_OVERLAP=1 STL_TC_DYN=30" "STL_FWD_OVERLAP=0"; do
  echo "$e $(env STL_LIB=$P $e timeout 300 python scripts/north_star.py 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["burst"]["stl_ms"],4), round(d["burst"]["cublas_ms"],4), round(d["burst"]["speedup"],3))')" >> $o
done; done
cat $o
