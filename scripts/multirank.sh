#!/bin/bash
# The multi-rank bench path on the one leased GPU: 2 ranks under torchrun, both on cuda:0,
# gloo (NCCL refuses two ranks on one device). Shows the DP step (g_w all-reduce on a side
# stream beside the g_x / g_ex decode) and the M-sharded 8192^3 forward run end to end.
mkdir -p gpurun_out
tag=${1:-multirank}
STL_BENCH_SAME_DEVICE=1 STL_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run \
  --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-t2t --no-cpu-baseline \
  > gpurun_out/${tag}.json 2> gpurun_out/${tag}.err
echo "rc=$?"
tail -c 1500 gpurun_out/${tag}.json; tail -5 gpurun_out/${tag}.err
