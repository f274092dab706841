#!/bin/bash
for rep in 1 2; do for v in 0 1; do
  SBT_DMMA_BB16=$v timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu --steps 10 > gpurun_out/ab_bb16_$v.json 2>&1
  echo "rep$rep bb16=$v $(grep -o '"value": [0-9.]*' gpurun_out/ab_bb16_$v.json | head -1) $(grep -o '"plain": {[^}]*}' gpurun_out/ab_bb16_$v.json | grep -o '"tflops": [0-9.]*') $(grep -o '"exceptional": {[^}]*}' gpurun_out/ab_bb16_$v.json | grep -o '"tflops": [0-9.]*')"
done; done
