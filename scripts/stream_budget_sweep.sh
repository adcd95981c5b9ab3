mkdir -p gpurun_out
{
for KB in 212 220 224; do for T in 0 512; do
  echo "KB=$KB T=$T"; STL_STREAM_SMEM_KB=$KB STL_STREAM_T=$T timeout 120 python scripts/transform_probe.py 2>&1 | tail -1 | cut -c60-230
done; done
} > gpurun_out/sweep2.log 2>&1
cat gpurun_out/sweep2.log
