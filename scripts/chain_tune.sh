#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/chain_tune.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for e in "STL_STREAM_NBUF=2" "STL_STREAM_T=256" "STL_STREAM_T=256 STL_STREAM_NBUF=3" "STL_STREAM_T=256 STL_STREAM_NBUF=4" "STL_STREAM_NBUF=2 STL_STREAM_SMEM_KB=222"; do
  echo "$e $(env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["remix_us"],1), round(d["fused_chain_ms"],4), round(d["unfused_ms"],4))')" >> $o
done
cat $o
