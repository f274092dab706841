#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or ritz or acc64 or factor" > gpurun_out/g5_parity_hooi.log 2>&1; tail -3 gpurun_out/g5_parity_hooi.log
timeout 300 python tools/hooi_trace.py > gpurun_out/g5_hooi_trace.txt 2>&1; head -16 gpurun_out/g5_hooi_trace.txt
SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_clock.so timeout 300 python tools/ritz_probe.py > gpurun_out/g5_ritz_probe.txt 2>&1; cat gpurun_out/g5_ritz_probe.txt
for g in 1 2 4; do
  SBT_TC_FLUSH_G=$g timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/g5_bench_hooi_g$g.json 2>&1; echo "G=$g"; grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*' gpurun_out/g5_bench_hooi_g$g.json | head -3
done
export SBTENSOR_BACKEND=b200 PYTHONPATH=$PWD/paper_1606_05696_b200/refhook:$PWD:$PWD/baseline/_ref NUMBA_CACHE_DIR=/tmp/numba_cache
(cd /tmp && timeout 120 python -u -m sbtensor.cli cases 2 3 --verify --dim 5 > $GRAFT_REPO_ROOT/gpurun_out/g5_cases.txt 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/gpurun_out/g5_cases.txt)
tail -5 gpurun_out/g5_cases.txt
unset SBTENSOR_BACKEND PYTHONPATH
timeout 600 python -m pytest tests/test_gpu_large.py -x -q -k "hooi" > gpurun_out/g5_large_hooi.log 2>&1; tail -3 gpurun_out/g5_large_hooi.log
