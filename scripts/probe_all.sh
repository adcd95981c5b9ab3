#!/bin/bash
# Quick A/B probe: GEMM micro-bench, fused vs unfused forward, transform variants.
mkdir -p gpurun_out
{
echo "=== gemm"; python scripts/gemm_bench.py
echo "=== fused"; python scripts/fused_probe.py
echo "=== fused72"; STL_FUSED_PAIRS=72 python scripts/fused_probe.py
echo "=== fused72 dbg"; STL_FUSED_DEBUG=1 STL_FUSED_PAIRS=72 python scripts/fused_probe.py 2>&1 | tail -8
echo "=== transforms"; python scripts/transform_probe.py
} > gpurun_out/probe_all.log 2>&1
cat gpurun_out/probe_all.log
