#!/bin/bash
mkdir -p gpurun_out
SBT_GA_DEBUG=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"w_kernel|z_kernel" -c 4 -o gpurun_out/g9_wz -f python tools/factor_bench.py > gpurun_out/g9_ncu.log 2>&1; tail -2 gpurun_out/g9_ncu.log
