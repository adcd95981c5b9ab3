#!/bin/bash
# the driver's round-end bench pair on one box: the default bench line and the reference arm
tag=${1:-r02c}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
tail -c 600 gpurun_out/bench_${tag}.err; tail -c 300 gpurun_out/bench_ref_${tag}.json
