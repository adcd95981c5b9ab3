#!/bin/bash
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -1
o=gpurun_out/dectf32_ab2.log; : > $o
for i in 1 2; do for e in STL_DEC_TF32=-1 STL_DEC_TF32=0; do
  echo "$e $(env $e timeout 300 python scripts/stream_tune.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["enc_us"], d["dec_us"], d["fwd_us"])')" >> $o
  echo "$e chain $(env STL_LIB=$PWD/paper_2503_12211_b200/libstl_b200_probe.so $e timeout 300 python scripts/bench_chain.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fused_chain_ms"], d["unfused_ms"], d["remix_us"])')" >> $o
done; done
cat $o
bash scripts/ab_step.sh ab_dectf32b "STL_DEC_TF32=-1" "STL_DEC_TF32=0" 2
