#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"w_kernel|z_kernel|ritz_kernel" -c 8 -o gpurun_out/g6_factor -f python tools/factor_probe.py > gpurun_out/g6_ncu.log 2>&1; tail -3 gpurun_out/g6_ncu.log
export SBTENSOR_BACKEND=b200 PYTHONPATH=$PWD/paper_1606_05696_b200/refhook:$PWD:$PWD/baseline/_ref NUMBA_CACHE_DIR=/tmp/numba_cache
(cd /tmp && timeout 120 python -u -m sbtensor.cli cases 2 3 --verify --dim 5 > $GRAFT_REPO_ROOT/gpurun_out/g6_cases.txt 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/gpurun_out/g6_cases.txt)
tail -2 gpurun_out/g6_cases.txt
unset SBTENSOR_BACKEND PYTHONPATH
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or ritz or acc64 or factor" > gpurun_out/g6_parity_hooi.log 2>&1; tail -3 gpurun_out/g6_parity_hooi.log
