#!/bin/bash
# tcgen05 decode (stl_stream_tc.cu) vs the mma.sync streaming decode: parity tests, then
# alternating A/B of the 8192^3 decode / forward (stream_tune.py) and the config-2 step.
# usage: scripts/dectc_ab.sh <tag> "<env A>" "<env B>" ...   (default: TC on vs off)
mkdir -p gpurun_out
tag=${1:-dectc_ab}; shift
vars=("$@"); [ ${#vars[@]} -eq 0 ] && vars=("STL_DEC_TC=1" "STL_DEC_TC=0")
o=gpurun_out/$tag.log; : > $o
timeout 900 python -m pytest tests/test_stream_transforms.py tests/test_parity_gpu.py -q -x 2>&1 | tail -3 >> $o
for e in "${vars[@]}"; do
  env STL_LIB=$PWD/paper_2503_12211_b200/libstl_b200_probe.so $e timeout 300 python -m pytest tests/test_stream_transforms.py -q -x -k "encode_decode_bf16" 2>&1 | tail -1 | sed "s/^/$e /" >> $o
done
for i in 1 2 3; do for e in "${vars[@]}"; do
  echo "$e $(env $e timeout 300 python scripts/stream_tune.py 2>&1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["enc_us"], d["dec_us"], d["fwd_us"], d["h"])')" >> $o
done; done
for i in 1 2; do for e in "${vars[@]}"; do
  env STL_LIB=$PWD/paper_2503_12211_b200/libstl_b200_probe.so $e timeout 300 python bench.py --steps 50 --warmup 10 --no-extras --no-cpu-baseline --no-t2t --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})" >> $o
done; done
timeout 300 python scripts/north_star.py 2>&1 | tail -1 >> $o
cat $o
