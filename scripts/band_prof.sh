#!/bin/bash
mkdir -p gpurun_out
tag=${1:-bandprof}
{
for v in "STL_BAND_NOSIDE=0" "STL_BAND_NOSIDE=3" "STL_BAND_NOSIDE=1" "STL_BAND_NOSIDE=2" "STL_BAND0_MB=3" "STL_BAND0_MB=5"; do
  echo "== $v"; env $v STL_BAND_PROFILE=1 ITERS=5 timeout 300 python scripts/probe_fwd.py 2>&1 | tail -4
done
echo "== noband"; STL_NOBAND=1 STL_PROFILE=1 ITERS=5 timeout 300 python scripts/probe_fwd.py 2>&1 | tail -2
} > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
