#!/bin/bash
mkdir -p gpurun_out
SBT_GA_DEBUG=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"w_kernel|z_kernel" -c 2 -o gpurun_out/g12_wz -f python tools/factor_bench.py > gpurun_out/g12_ncu.log 2>&1; tail -1 gpurun_out/g12_ncu.log
