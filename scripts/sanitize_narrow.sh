#!/bin/bash
# memcheck / synccheck on the tcgen05 encode / decode with multi-row (narrow-matrix) units
mkdir -p gpurun_out
{
for tool in memcheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 \
    python -m pytest tests/test_stream_transforms.py -m gpu -q -x -p no:cacheprovider \
    -k "encode_decode_bf16 and (24-36-256 or 20-148-256 or 24-128-512 or 5-52-512)" 2>&1 | grep -vE "^\.+ *\[" | tail -4
  echo "rc=${PIPESTATUS[0]}"
done
} > gpurun_out/sanitize_narrow.log 2>&1
cat gpurun_out/sanitize_narrow.log
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
