#!/bin/bash
mkdir -p gpurun_out
{ timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or layer or batched" 2>&1 | tail -2
for pf in 0 1; do echo "evict=$pf"; STL_GEMM_EVICT=$pf STL_GEMM_DEBUG=1 python scripts/transform_probe.py 2>&1 | grep "gemm dbg" | tail -3
STL_GEMM_EVICT=$pf python scripts/gemm_bench.py
STL_GEMM_EVICT=$pf timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['vs_cublas']['speedup'], d['north_star_fwd_8192']['speedup'], d['roofline']['achieved'], {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})"
done
} > gpurun_out/gemm_sweep.log 2>&1
cat gpurun_out/gemm_sweep.log
