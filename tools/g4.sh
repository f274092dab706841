#!/bin/bash
# HOOI rework: factor-update kernels, acc64 core product, C4 parity, breakdown
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or ritz or acc64 or factor" > gpurun_out/g4_parity_hooi.log 2>&1; tail -5 gpurun_out/g4_parity_hooi.log
timeout 600 python -m pytest tests/test_gpu_large.py -x -q -k "hooi" > gpurun_out/g4_large_hooi.log 2>&1; tail -5 gpurun_out/g4_large_hooi.log
timeout 300 python tools/hooi_trace.py > gpurun_out/g4_hooi_trace.txt 2>&1; cat gpurun_out/g4_hooi_trace.txt | head -40
timeout 300 python tools/ritz_probe.py > gpurun_out/g4_ritz_probe.txt 2>&1; cat gpurun_out/g4_ritz_probe.txt
timeout 400 python bench.py --config hooi > gpurun_out/g4_bench_hooi.json 2> gpurun_out/g4_bench_hooi.err; tail -c 600 gpurun_out/g4_bench_hooi.json
SBT_TC_FLUSH=0 timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/g4_bench_hooi_noflush.json 2>&1; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9., ]*' gpurun_out/g4_bench_hooi_noflush.json | head -3
timeout 900 python -m pytest tests/test_refcli.py -x -q > gpurun_out/g4_refcli.log 2>&1; tail -5 gpurun_out/g4_refcli.log
