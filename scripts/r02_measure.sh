#!/bin/bash
# round-2 evidence on one box: GPU suite + smoke, the default bench line, the reference arm,
# ncu launch list + full sets (config-2 step and the 8192^3 forward's transforms)
tag=${1:-r02b}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh gt_${tag}
timeout 1500 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
bash scripts/ncu_capture.sh $tag
bash scripts/ncu_fwd8192.sh ${tag}_fwd8192
tail -c 2500 gpurun_out/bench_${tag}.json; echo; tail -c 800 gpurun_out/bench_ref_${tag}.json
