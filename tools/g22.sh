#!/bin/bash
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ritz or factor or hooi" 2>&1 | tail -2
SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_clock.so timeout 300 python tools/ritz_probe.py
timeout 300 python tools/hooi_trace.py 2>&1 | grep -v Warn | sed -n 2,9p
timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/g22_bench_hooi.json 2>&1; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*' gpurun_out/g22_bench_hooi.json | head -3
echo "== fp64 sweep BK16 vs BK32"
timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu > gpurun_out/g22_sweep_bk16.json 2>&1; grep -o '"value": [0-9.]*' gpurun_out/g22_sweep_bk16.json | head -1; grep -o '"plain": {[^}]*}\|"exceptional": {[^}]*}' gpurun_out/g22_sweep_bk16.json
SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_bk32.so timeout 300 python bench.py --dtype f64 --no-e2e --no-cpu > gpurun_out/g22_sweep_bk32.json 2>&1; grep -o '"value": [0-9.]*' gpurun_out/g22_sweep_bk32.json | head -1; grep -o '"plain": {[^}]*}\|"exceptional": {[^}]*}' gpurun_out/g22_sweep_bk32.json
SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_bk32.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f64 or dmma or 36" 2>&1 | tail -2
