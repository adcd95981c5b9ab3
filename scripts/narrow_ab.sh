#!/bin/bash
# tcgen05 encode / decode on narrow matrices (units of R whole tile rows): tests, then the
# T2T-ViT-7 training step with the narrow path on / off (STL_TC_NARROW probe via STL_ENC_TC /
# STL_DEC_TC off as the baseline)
mkdir -p gpurun_out
o=gpurun_out/narrow_ab.log; : > $o
timeout 1200 python -m pytest tests/test_stream_transforms.py tests/test_tc_transforms.py tests/test_t2t_vit.py tests/test_parity_gpu.py -q -x 2>&1 | tail -2 >> $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for i in 1 2; do for e in "STL_X=1" "STL_ENC_TC=0 STL_DEC_TC=0"; do
  echo "$e $(env STL_LIB=$P $e timeout 600 python scripts/bench_t2t.py 2>/dev/null | tail -1 | cut -c1-300)" >> $o
done; done
cat $o
