#!/bin/bash
# round-end evidence: ncu capture (launch list + full sets), default bench line, reference arm
tag=${1:-r01e}
mkdir -p gpurun_out
bash scripts/ncu_capture.sh $tag
timeout 1200 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
tail -c 3000 gpurun_out/bench_${tag}.json; echo; tail -c 1500 gpurun_out/bench_ref_${tag}.json
