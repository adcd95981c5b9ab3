#!/bin/bash
# interleaved A/B of probe switches: bash scripts/ab.sh <tag> "<VARIANTS>" (WORK, ROUNDS env)
mkdir -p gpurun_out
tag=${1:-ab}
export STL_LIB=paper_2503_12211_b200/libstl_b200_probe.so
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/${tag}_clocks.csv &
SMI=$!
VARIANTS="$2" timeout 1200 python scripts/ab_interleaved.py > gpurun_out/${tag}.log 2>&1
kill $SMI
cat gpurun_out/${tag}.log
python - <<PY
import csv
rows = list(csv.reader(open("gpurun_out/${tag}_clocks.csv")))[1:]
mhz = sorted(int(r[0].split()[0]) for r in rows if r and r[0].strip()[0].isdigit())
pw = sorted(float(r[1].split()[0]) for r in rows if r and r[1].strip()[0].isdigit())
print("clock samples", len(mhz), "median MHz", mhz[len(mhz)//2], "min", mhz[0], "power median", pw[len(pw)//2], "max", pw[-1])
PY
