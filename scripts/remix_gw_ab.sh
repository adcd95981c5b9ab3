#!/bin/bash
# k_remix_tc epilogue width: 4 vs 8 warps per group (STL_REMIX_TC_GW), f1 chain bench + tests
mkdir -p gpurun_out
o=gpurun_out/remix_gw_ab.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
STL_LIB=$P STL_REMIX_TC_GW=8 timeout 900 python -m pytest tests/test_tc_transforms.py -q -x -k "remix" 2>&1 | tail -2 >> $o
for i in 1 2 3; do for e in "STL_REMIX_TC_GW=4" "STL_REMIX_TC_GW=8"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4))" >> $o
done; done
cat $o
