#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or ritz or acc64 or factor" > gpurun_out/g7_parity_hooi.log 2>&1; tail -3 gpurun_out/g7_parity_hooi.log
timeout 300 python tools/hooi_trace.py > gpurun_out/g7_hooi_trace.txt 2>&1; head -14 gpurun_out/g7_hooi_trace.txt
for g in 4 8; do
  SBT_TC_FLUSH_G=$g timeout 300 python tools/hooi_trace.py > gpurun_out/g7_hooi_trace_g$g.txt 2>&1; echo "G=$g"; head -5 gpurun_out/g7_hooi_trace_g$g.txt | tail -3
  SBT_TC_FLUSH_G=$g timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/g7_bench_hooi_g$g.json 2>&1; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*' gpurun_out/g7_bench_hooi_g$g.json | head -3
done
SBT_TC_FLUSH_G=8 timeout 600 python -m pytest tests/test_gpu_large.py -x -q -k "hooi" > gpurun_out/g7_large_hooi_g8.log 2>&1; tail -3 gpurun_out/g7_large_hooi_g8.log
