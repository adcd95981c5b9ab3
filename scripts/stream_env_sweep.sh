#!/bin/bash
# streaming-transform launch parameters on the config-2 step (unit size T, ring stages)
mkdir -p gpurun_out
{
for T in 256 512; do for ST in 4 6 8 12 16; do
  echo "T=$T stages=$ST"; STL_STREAM_T=$T STL_STREAM_STAGES=$ST timeout 120 python scripts/transform_probe.py 2>&1 | tail -1 | cut -c1-230
done; done
echo default; timeout 120 python scripts/transform_probe.py 2>&1 | tail -1 | cut -c1-230
} > gpurun_out/stream_env_sweep.log 2>&1
cat gpurun_out/stream_env_sweep.log
