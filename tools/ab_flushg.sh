#!/bin/bash
for g in 4 8; do
  SBT_TC_FLUSH_G=$g timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/ab_g$g.json 2>&1
  echo "G=$g $(grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*' gpurun_out/ab_g$g.json | head -2 | tr '\n' ' ')"
done
