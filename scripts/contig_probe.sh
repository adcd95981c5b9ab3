#!/bin/bash
# data-movement floor of the 8192^3 encode / decode (NOCOMPUTE) with the planes moved as TMA
# boxes (current), per-plane bulk copies, or one contiguous bulk copy per unit (blocked layout)
o=gpurun_out/contig_probe.log; : > $o
run() { env STL_STREAM_NOCOMPUTE=1 "$@" timeout 300 python scripts/stream_tune.py 2>&1 >> $o; }
run STL_X=box
run STL_BULK_IN=1 STL_BULK_OUT=1
run STL_BULK_IN=1 STL_BULK_OUT=1 STL_PROBE_CONTIG=1
run STL_X=box
run STL_BULK_IN=1 STL_BULK_OUT=1 STL_PROBE_CONTIG=1
cat $o
run2() { env "$@" timeout 300 python scripts/stream_tune.py 2>&1 >> $o; }
run2 STL_X=box_compute
run2 STL_BULK_IN=1 STL_BULK_OUT=1
