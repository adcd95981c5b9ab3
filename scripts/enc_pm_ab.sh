#!/bin/bash
# plane-major output box for the tcgen05 encode (STL_ENC_PM): tests with it on, then A/B
mkdir -p gpurun_out
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
o=gpurun_out/enc_pm_ab.log; : > $o
STL_LIB=$P STL_ENC_PM=1 timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_tc_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -2 >> $o
bash scripts/dectc_ab.sh enc_pm_ab2 "STL_ENC_PM=1" "STL_ENC_PM=0" | tail -12 >> $o
cat $o
