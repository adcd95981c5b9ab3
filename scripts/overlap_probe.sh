#!/bin/bash
# co-residency probe variants (scripts/overlap_probe.py), one process each
mkdir -p gpurun_out
o=gpurun_out/overlap_probe2.log
: > $o
export STL_SMEM_MAX_CARVEOUT=1
STL_GEMM_STAGES=4 STL_STREAM_CW=8 STL_STREAM_SMEM_KB=60 timeout 120 python scripts/overlap_probe.py >> $o 2>&1
STL_GEMM_STAGES=4 STL_STREAM_CW=8 STL_STREAM_SMEM_KB=48 timeout 120 python scripts/overlap_probe.py >> $o 2>&1
STL_GEMM_STAGES=4 STL_STREAM_CW=8 STL_STREAM_SMEM_KB=36 timeout 120 python scripts/overlap_probe.py >> $o 2>&1
STL_GEMM_STAGES=4 timeout 120 python scripts/overlap_probe.py >> $o 2>&1
timeout 120 python scripts/overlap_probe.py >> $o 2>&1
cat $o
