#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on this round's new kernels: t = 2 streaming
# transforms, the remix (bulk-store output, in-kernel composite), the TF32 bf16-plane decode
mkdir -p gpurun_out
SEL_T2='t2 and (64-2048-24 or 130-72-3 or 6-520-49)'
SEL_CHAIN='chain_bf16_streamed_remix and (13-256 or 24-512)'
SEL_DEC='encode_decode_bf16 and (24-36-256 or 24-64-2304) or layer_fwd_bwd_formats and 24-bf16'
{
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider -k "$SEL_T2 or $SEL_DEC" 2>&1 | tail -3
  echo "rc=${PIPESTATUS[0]}"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "$SEL_CHAIN" 2>&1 | tail -3
  echo "rc=${PIPESTATUS[0]}"
done
} > gpurun_out/sanitize_r02.log 2>&1
cat gpurun_out/sanitize_r02.log
