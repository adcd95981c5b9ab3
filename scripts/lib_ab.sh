#!/bin/bash
# interleaved A/B of two product library builds on the config-2 step and the 8192^3 forward
o=gpurun_out/lib_ab.log; : > $o
for i in 1 2 3; do
  for L in $PWD/paper_2503_12211_b200/libstl_b200.so $PWD/build_ab/old_prod.so; do
    s=$(STL_LIB=$L timeout 300 python bench.py --steps 50 --warmup 10 --no-extras --no-cpu-baseline --no-t2t --no-sweep 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
    f=$(STL_LIB=$L timeout 300 python scripts/north_star.py 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['burst']['stl_ms'],4), round(d['burst']['speedup'],3))")
    echo "$(basename $L) step=$s fwd8192=$f" >> $o
  done
done
cat $o
