#!/bin/bash
export PYTHONDONTWRITEBYTECODE=1
for v in 1 0; do
  SBT_DMMA_BB16=$v timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu --steps 5 > gpurun_out/ab_bb16_$v.json 2>&1
  echo "bb16=$v $(grep -o '"value": [0-9.]*' gpurun_out/ab_bb16_$v.json | head -1) $(grep -o '"exceptional": {[^}]*}' gpurun_out/ab_bb16_$v.json)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "f64 or float64 or exceptional or 3.4 or 3.6 or 4.4 or 4.6 or 5.4 or 5.6 or 6.4 or 6.6 or ragged or bb" 2>&1 | tail -1
