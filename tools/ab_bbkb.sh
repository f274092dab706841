#!/bin/bash
export PYTHONDONTWRITEBYTECODE=1
SBT_TC_BB_KB=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "3.4 or 3.6 or 4.4 or 4.6 or 5.4 or 5.6 or 6.4 or 6.6 or exceptional or ragged or bb" 2>&1 | tail -1
bash tools/ab_env.sh "--dtype f32 --no-e2e --no-cpu --steps 10" SBT_TC_BB_KB 32 16 2
