#!/bin/bash
mkdir -p gpurun_out
tag=${1:-band}
{
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "banded or slice_gemm_wide or full_size_row_slab" 2>&1 | tail -5
for v in "STL_NOBAND=1" "STL_NOBAND=0" "STL_BAND0_MB=3" "STL_BAND0_MB=5" "STL_BAND_REV=0" "STL_GEMM_LAG=0"; do
  env $v timeout 300 python scripts/probe_fwd.py
done
STL_NOBAND=1 STL_GEMM_NOWIDE=1 timeout 300 python scripts/probe_fwd.py
} > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
