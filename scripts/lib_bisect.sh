#!/bin/bash
o=gpurun_out/lib_bisect.log; : > $o
for i in 1 2; do
  for L in build_ab/old_prod.so build_ab/prod_d366371.so build_ab/prod_9949d05.so paper_2503_12211_b200/libstl_b200.so; do
    s=$(STL_LIB=$PWD/$L timeout 300 python bench.py --steps 50 --warmup 10 --no-extras --no-cpu-baseline --no-t2t --no-sweep 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v['ms_per_step']*1e3,1) for k,v in d['kernels'].items()})")
    echo "$(basename $L) $s" >> $o
  done
done
cat $o
