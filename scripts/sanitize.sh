#!/bin/bash
# compute-sanitizer memcheck / synccheck over a representative subset of the GPU parity tests
mkdir -p gpurun_out
SEL_STREAM='encode_decode_bf16 and (24-36-256 or 5-8-4096) or layer_fwd_bwd_formats and (13-f24 or 24-bf16)'
SEL_PAR='slice_gemm_tc_layouts and (shape1 or shape4) or stl_batched_bf16 and 1024-1024-1024-4-24'
{
for tool in memcheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider -k "$SEL_STREAM" 2>&1 | tail -4
  echo "rc=${PIPESTATUS[0]}"
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "$SEL_PAR" 2>&1 | tail -4
  echo "rc=${PIPESTATUS[0]}"
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_t2t_vit.py -m gpu -q -x -p no:cacheprovider -k "token_kernels" 2>&1 | tail -4
  echo "rc=${PIPESTATUS[0]}"
done
} > gpurun_out/sanitize.log 2>&1
cat gpurun_out/sanitize.log
