#!/bin/bash
# config-2 step + north-star forward: default build vs probe variants (short bench legs)
mkdir -p gpurun_out
tag=${1:-step}
export TAGN=$tag
P=paper_2503_12211_b200/libstl_b200_probe.so
{
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1 > gpurun_out/${tag}_bench.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/%s_bench.json" % __import__("os").environ["TAGN"]))
print(d["ms_per_step"], d["vs_cublas"], d["north_star_fwd_8192"])
for k, v in d["kernels"].items(): print(k, v)
PY
for v in "STL_GEMM_WIDEF32=1" "STL_GEMM_WIDEF32=1 STL_GEMM_LAG=0" "STL_GEMM_NOWIDE=1"; do
  echo "== $v"; env STL_LIB=$P $v timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-t2t 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['vs_cublas']['speedup'], d['north_star_fwd_8192']['stl_ms'], d['kernels']['slice_gemm_tcgen05'])"
done
} > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
