#!/bin/bash
# wide-tile slice GEMM: parity tests + timing at the north-star shape (lag / split variants)
mkdir -p gpurun_out
export STL_LIB=paper_2503_12211_b200/libstl_b200_probe.so  # STL_* switches: probe build
tag=${1:-wide}
{
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "slice_gemm or layer_backward or stl_batched or full_size" 2>&1 | tail -5
for v in "STL_GEMM_NOWIDE=1" "STL_GEMM_LAG=0" "STL_GEMM_LAG=1" "STL_GEMM_LAG=2" "STL_GEMM_LAG=2 STL_GEMM_NOSPLIT=1" "STL_GEMM_LAG=2 STL_GEMM_NOSTORE=1"; do
  echo "== $v"; env $v timeout 300 python scripts/probe_gemm_l2.py stl
done
timeout 300 python scripts/probe_gemm_l2.py bmm
timeout 300 python scripts/gemm_bench.py cfg2_fwd cfg2_gu cfg2_gw n8192
STL_GEMM_NOWIDE=1 timeout 300 python scripts/gemm_bench.py cfg2_fwd cfg2_gu cfg2_gw n8192
} > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
