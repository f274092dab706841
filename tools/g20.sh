#!/bin/bash
timeout 300 python tools/hooi_trace.py 2>&1 | grep -v Warn | sed -n 1,12p
timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/g20_bench_hooi.json 2>&1; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*' gpurun_out/g20_bench_hooi.json | head -3
