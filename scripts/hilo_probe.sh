#!/bin/bash
o=gpurun_out/hilo_probe.log; : > $o
for e in STL_HILO=1 STL_HILO=0 STL_HILO=1 STL_HILO=0; do env $e timeout 300 python scripts/stream_tune.py >> $o 2>&1; done
python3 -c "
import re
for l in open('$o'):
    m=re.findall(r'\"(enc_us|dec_us|fwd_us)\": ([0-9.]+)', l); e=re.findall(r'\"(STL_HILO)\": \"([^\"]*)\"', l); print(e, m)"
