#!/bin/bash
mkdir -p gpurun_out
for d in 1 2 0; do SBT_GA_DEBUG=$d timeout 120 python tools/factor_bench.py; done > gpurun_out/g8_factor_bench.txt 2>&1
cat gpurun_out/g8_factor_bench.txt
