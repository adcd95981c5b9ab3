#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/evict_ab.log; : > $o
run() { env "$@" timeout 300 python scripts/stream_tune.py >> $o 2>&1; }
for i in 1 2; do
run STL_X=base
run STL_GEMM_EVICT_FIRST=1
run STL_DEC_EVICT_FIRST=1
run STL_GEMM_EVICT_FIRST=1 STL_DEC_EVICT_FIRST=1
done
cat $o
