#!/bin/bash
for rep in 1 2; do for lib in libsbt200 libsbt200_bk32s2; do
  SBT_LIB=$PWD/paper_1606_05696_b200/lib/$lib.so timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu --steps 10 > gpurun_out/ab_bk_$lib.json 2>&1
  echo "rep$rep $lib $(grep -o '"value": [0-9.]*' gpurun_out/ab_bk_$lib.json | head -1) $(grep -o '"plain": {[^}]*}' gpurun_out/ab_bk_$lib.json | grep -o '"tflops": [0-9.]*') $(grep -o '"exceptional": {[^}]*}' gpurun_out/ab_bk_$lib.json | grep -o '"tflops": [0-9.]*')"
done; done
