#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/l2_handoff2.log
: > $o
run() { env "$@" timeout 300 python scripts/l2_handoff.py >> $o 2>&1; sleep 5; }
run STL_L2_KEEP_MB=0
run STL_L2_KEEP_MB=48 STL_L2_GEMM=0
run STL_L2_KEEP_MB=48 STL_L2_ENC=0 STL_L2_DISCARD=0
run STL_L2_KEEP_MB=48 STL_L2_ENC=0
run STL_L2_KEEP_MB=0
run STL_L2_KEEP_MB=24 STL_L2_ENC=0
run STL_L2_KEEP_MB=24 STL_L2_GEMM=0
cat $o
