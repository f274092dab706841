#!/bin/bash
# fp64 DMMA default-tile validation: parity subset + the fp64 bench lines
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_conventional.py -q -x -k "f64 or dmma or 36 or c1 or hooi or float64" 2>&1 | tail -1
for c in "sweep_f64" "c1 --config c1" "order4_f64 --config order4 --dtype f64" "hooi_f64 --config hooi --dtype f64 --no-e2e"; do
  set -- $c; name=$1; shift
  timeout 400 python bench.py "$@" > gpurun_out/chk_$name.json 2>&1
  echo "$name: $(grep -o '"value": [0-9.]*' gpurun_out/chk_$name.json | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/chk_$name.json | head -1) $(grep -o '"ms_per_iteration": [0-9.]*' gpurun_out/chk_$name.json)"
done
