#!/bin/bash
for w in 0 8; do
  SBT_DMMA_WARPS=$w timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu --steps 5 > gpurun_out/ab_bbw$w.json 2>&1
  echo "warps=$w $(grep -o '"exceptional": {[^}]*}' gpurun_out/ab_bbw$w.json)"
done
