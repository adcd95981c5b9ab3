#!/bin/bash
# grouped backward GEMM: gpu tests + A/B of the config-2 step (STL_GEMM_NOGROUP=1 = two launches)
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for i in 1 2 3; do
  echo "group"; timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-300
  echo "nogroup"; STL_GEMM_NOGROUP=1 timeout 300 python scripts/transform_probe.py | tail -1 | cut -c1-300
done
STL_GEMM_DEBUG=1 timeout 300 python scripts/transform_probe.py 2>&1 | grep "gemm dbg" | sort | uniq -c | head
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1
  STL_GEMM_NOGROUP=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1
done
} > gpurun_out/group_ab.log 2>&1
cat gpurun_out/group_ab.log
