#!/bin/bash
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for e in "STL_BULK_PLANES=1" "STL_BULK_PLANES=0" "STL_BULK_PLANES=1" "STL_BULK_PLANES=0"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4), d['rel_diff_fused_vs_unfused'])"
done
env STL_LIB=$P STL_BULK_PLANES=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "chain" 2>&1 | tail -1
