#!/bin/bash
# k_remix_tc tuning: staging buffers / schedule variants on the f1 chain bench + one ncu capture
mkdir -p gpurun_out
o=gpurun_out/${1:-remix_tune}.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for i in 1 2; do for e in "STL_REMIX_TC_NBUF=2" "STL_REMIX_TC_NBUF=3" "STL_TC_DYN=0" "STL_TC_DYN=-1" "STL_TC_DYN=24"; do
  env STL_LIB=$P $e timeout 300 python scripts/bench_chain.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['remix_us'],1), round(d['fused_chain_ms'],4), round(d['unfused_ms'],4))" >> $o
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_remix_tc -s 3 -c 1 -o gpurun_out/ncu_remix python scripts/bench_chain.py > gpurun_out/ncu_remix.log 2>&1
cat $o
