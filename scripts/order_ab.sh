#!/bin/bash
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -1
bash scripts/ab_step.sh ab_order "STL_GEMM_ORDER=1" "STL_GEMM_ORDER=0" 3
