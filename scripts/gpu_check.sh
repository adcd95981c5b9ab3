#!/bin/bash
# full GPU test suite + smoke + a short bench line (clocks sampled in the timed region)
mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['clocks'], d['roofline']['frac'], d['north_star_fwd_8192']['speedup'], d['vs_cublas']['speedup'])"
} > gpurun_out/gpu_check.log 2>&1
cat gpurun_out/gpu_check.log
