#!/bin/bash
# ncu --set full of the config-2 step's two tc2 launches (forward, grouped backward) + launch list
mkdir -p gpurun_out
tag=${1:-stepgemm}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 6 -c 2 \
  -o gpurun_out/${tag} python scripts/transform_probe.py > gpurun_out/${tag}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv \
  --log-file gpurun_out/${tag}_launches.csv python scripts/transform_probe.py > /dev/null 2>&1
ls -la gpurun_out | grep ${tag}
