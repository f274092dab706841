#!/bin/bash
# HOOI parity + timing check
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "hooi or factor or acc64 or narrow or long" 2>&1 | tail -1
timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/chk_hooi.json 2>&1; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*\|"frac": [0-9.]*' gpurun_out/chk_hooi.json | head -3
