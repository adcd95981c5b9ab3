#!/bin/bash
# tcgen05 remix (k_remix_tc) vs the mma.sync streaming remix: new TC tests, then the f1 chain
# bench (3 bf16 layers at 8192^3) alternating
mkdir -p gpurun_out
o=gpurun_out/${1:-remix_tc_ab}.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
timeout 900 python -m pytest tests/test_tc_transforms.py tests/test_parity_gpu.py -q -x -k "tc_ or chain" 2>&1 | tail -3 >> $o
for i in 1 2 3; do for e in "STL_REMIX_TC=1" "STL_REMIX_TC=0"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4), d['rel_diff_fused_vs_unfused'])" >> $o
done; done
cat $o
