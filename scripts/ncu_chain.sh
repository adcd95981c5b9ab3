#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_stream<\(int\)4" -s 2 -c 1 -o gpurun_out/${1:-chain}_remix python scripts/bench_chain.py > gpurun_out/${1:-chain}_remix.log 2>&1
tail -3 gpurun_out/${1:-chain}_remix.log
