#!/bin/bash
# hybrid multicast schedule (STL_GEMM_MC=3) vs pair-only clusters: checks + micro-bench + step
mkdir -p gpurun_out
{
for mc in 3 1; do STL_GEMM_MC=$mc timeout 120 python scripts/gemm_check.py; done
STL_GEMM_MC=3 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or layer or batched or f24 or backward or forward" 2>&1 | tail -2
for i in 1 2; do
for mc in 3 1; do
  echo "== MC=$mc"
  STL_GEMM_MC=$mc timeout 120 python scripts/gemm_bench.py | cut -c1-90
  STL_GEMM_MC=$mc timeout 120 python scripts/transform_probe.py | tail -1 | cut -c1-250
done
done
for sh in 0.06 0.08 0.12; do echo "share $sh"; STL_GEMM_MC=3 STL_GEMM_HYBRID_SHARE=$sh timeout 120 python scripts/gemm_bench.py cfg2_fwd n8192 | cut -c1-90; done
for mc in 3 1; do STL_GEMM_MC=$mc timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MC', $mc, d['ms_per_step'], d['north_star_fwd_8192']['stl_ms'], d['north_star_fwd_8192']['speedup'], d['roofline']['achieved'])"; done
} > gpurun_out/mc_ab.log 2>&1
cat gpurun_out/mc_ab.log
