#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or ritz or acc64 or factor" > gpurun_out/g10_parity_hooi.log 2>&1; tail -3 gpurun_out/g10_parity_hooi.log
for d in 1 2 0; do SBT_GA_DEBUG=$d timeout 120 python tools/factor_bench.py; done > gpurun_out/g10_factor_bench.txt 2>&1
cat gpurun_out/g10_factor_bench.txt
