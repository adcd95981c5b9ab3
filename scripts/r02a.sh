bash scripts/gpu_tests.sh gt3
bash scripts/multirank.sh multirank_r02
timeout 900 python bench.py --steps 30 --warmup 5 --no-t2t > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; tail -c 4000 gpurun_out/bench_r02a.json
