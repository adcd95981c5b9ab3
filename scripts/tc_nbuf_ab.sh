#!/bin/bash
# staging-buffer counts of the tcgen05 encode / decode with the dynamic tail (8192^3 + config 2)
mkdir -p gpurun_out
bash scripts/dectc_ab.sh tc_nbuf_ab "STL_TC=default" "STL_ENC_TC_NBUF=3" "STL_DEC_TC_NBUF=2" "STL_ENC_TC_NBUF=3 STL_DEC_TC_NBUF=4"
