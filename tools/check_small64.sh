#!/bin/bash
# fp32 n=64 batched: mma.sync 3xTF32 kernel vs the FFMA kernel
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "small" 2>&1 | tail -1
SBT_SMALL64_MMA=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "small64" 2>&1 | tail -1
for v in 1 0; do
  SBT_SMALL64_MMA=$v timeout 300 python bench.py --config small --dtype f32 --no-e2e --no-cpu > gpurun_out/chk_small_mma$v.json 2>&1
  echo "mma=$v: $(grep -o '"n": 64, "batch": [0-9]*, "ms": [0-9.]*, "kernel": "[a-z0-9_]*", "gflops": [0-9.]*, "hbm_gbs": [0-9.]*, "frac_of_measured_hbm": [0-9.]*' gpurun_out/chk_small_mma$v.json)"
done
