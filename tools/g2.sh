#!/bin/bash
# round-2 validation: flush-mode parity at the BASELINE configs, new bench lines,
# HOOI breakdown, the reference suite against the b200 backend, 2 ranks on 1 GPU
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests/test_gpu_large.py -x -q -k "hooi or c1 or 1.1 or 6.4 or 3.6" > gpurun_out/g2_large_subset.log 2>&1; tail -3 gpurun_out/g2_large_subset.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hooi or narrow or skinny or fold or long" > gpurun_out/g2_parity_subset.log 2>&1; tail -3 gpurun_out/g2_parity_subset.log
timeout 300 python tools/hooi_trace.py > gpurun_out/g2_hooi_trace.txt 2>&1
timeout 300 python tools/ritz_probe.py > gpurun_out/g2_ritz_probe.txt 2>&1
timeout 400 python bench.py > gpurun_out/g2_bench_default.json 2> gpurun_out/g2_bench_default.err
timeout 300 python bench.py --config c1 > gpurun_out/g2_bench_c1.json 2> gpurun_out/g2_bench_c1.err
timeout 400 python bench.py --config hooi > gpurun_out/g2_bench_hooi.json 2> gpurun_out/g2_bench_hooi.err
SBT_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --config c1 --no-e2e --steps 3 > gpurun_out/g2_bench_c1_2ranks.json 2> gpurun_out/g2_bench_c1_2ranks.err
timeout 900 bash tools/run_ref_suite.sh > gpurun_out/g2_ref_suite.log 2>&1; tail -5 gpurun_out/g2_ref_suite.log
