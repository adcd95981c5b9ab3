#!/bin/bash
o=gpurun_out/tf32_ab3.log; : > $o
P=$PWD/paper_2503_12211_b200/libstl_b200_probe.so
for i in 1 2 3; do
  for e in STL_DEC_TF32=-1 STL_DEC_TF32=0 STL_DEC_TF32=2; do
    s=$(env STL_LIB=$P $e timeout 300 python bench.py --steps 50 --warmup 10 --no-extras --no-cpu-baseline --no-t2t --no-sweep 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})")
    f=$(env STL_LIB=$P $e timeout 300 python scripts/north_star.py 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['burst']['stl_ms'],4))")
    echo "$e step=$s fwd=$f" >> $o
  done
done
cat $o
