#!/bin/bash
mkdir -p gpurun_out
o=gpurun_out/${1:-stream_tune}.log
: > $o
run() { env "$@" timeout 300 python scripts/stream_tune.py >> $o 2>&1; }
run STL_STREAM_NBUF=2
run STL_STREAM_NBUF=3
run STL_STREAM_NBUF=2 STL_PDL=0
run STL_STREAM_NBUF=3 STL_PDL=0
cat $o
