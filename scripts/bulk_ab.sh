#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -1
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for e in "STL_X=1" "STL_BULK_IN=1" "STL_BULK_OUT=0" "STL_X=1" "STL_BULK_IN=1"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4))"
done
env STL_LIB=$P timeout 300 python scripts/stream_tune.py | cut -c1-200
