#!/bin/bash
# full GPU test suite + smoke (round-end equivalent), log under gpurun_out/
mkdir -p gpurun_out
tag=${1:-gputests}
{
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
} > gpurun_out/${tag}.log 2>&1
cat gpurun_out/${tag}.log
