#!/bin/bash
# A/B a variant library build on one bench config: ab_lib.sh "<bench args>" <variant .so name> [reps]
args=$1; var=$2; reps=${3:-2}
for rep in $(seq 1 $reps); do for lib in libsbt200 $var; do
  SBT_LIB=$PWD/paper_1606_05696_b200/lib/$lib.so timeout 400 python bench.py $args > gpurun_out/ab_lib.json 2>&1
  echo "rep$rep $lib $(grep -o '"value": [0-9.]*' gpurun_out/ab_lib.json | head -1) $(grep -o '"ms_per_iteration": [0-9.]*\|"hooi_paths": {[^}]*}\|"fit_history": \[[0-9.]*' gpurun_out/ab_lib.json | tr '\n' ' ')"
done; done
