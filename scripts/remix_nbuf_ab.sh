#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/remix_nbuf_ab.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for i in 1 2 3; do for e in "STL_REMIX_TC_NBUF=2" "STL_REMIX_TC_NBUF=3" "STL_REMIX_TC_NBUF=4"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4))" >> $o
done; done
cat $o
