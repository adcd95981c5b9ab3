#!/bin/bash
# compute-sanitizer racecheck (shared-memory hazards) + memcheck on the newer paths
mkdir -p gpurun_out
{
echo "== racecheck stream"
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --target-processes all --error-exitcode 9 \
  python -m pytest tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider -k "encode_decode_bf16 and 24-36-256 or layer_fwd_bwd_formats and 13-bf16" 2>&1 | tail -5
echo "rc=${PIPESTATUS[0]}"
echo "== racecheck tokens"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --target-processes all --error-exitcode 9 \
  python -m pytest tests/test_t2t_vit.py -m gpu -q -x -p no:cacheprovider -k "token_kernels" 2>&1 | tail -5
echo "rc=${PIPESTATUS[0]}"
echo "== memcheck gemm/formats"
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 \
  python -m pytest tests/test_parity_gpu.py tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider -k "inference or layer_fwd_bwd_formats or slice_gemm_tc_layouts and shape2" 2>&1 | tail -5
echo "rc=${PIPESTATUS[0]}"
} > gpurun_out/racecheck.log 2>&1
cat gpurun_out/racecheck.log
