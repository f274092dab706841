#!/bin/bash
# A/B of the fp64 DMMA tile configurations on the fp64 sweep (n = 128 / 256 / 512)
for n in 256 128 512; do
  for bn in 128 64; do
    SBT_DMMA_BN=$bn timeout 300 python bench.py --dtype f64 --n $n --no-e2e --no-cpu --steps 5 > gpurun_out/ab_dmma_bn${bn}_n$n.json 2>&1
    echo "n=$n BN=$bn: $(grep -o '"value": [0-9.]*' gpurun_out/ab_dmma_bn${bn}_n$n.json | head -1) $(grep -o '"plain": {[^}]*}' gpurun_out/ab_dmma_bn${bn}_n$n.json) $(grep -o '"exceptional": {[^}]*}' gpurun_out/ab_dmma_bn${bn}_n$n.json)"
  done
done
SBT_DMMA_BN=64 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "f64 or dmma or 36 or c1" 2>&1 | tail -1
