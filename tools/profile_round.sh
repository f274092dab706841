#!/bin/bash
# ncu captures of the dominant kernels at the bench configuration + launch list.
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o gpurun_out/prof_pair_1.3_n256 -f python tools/case_single.py 1.3 256 f32 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o gpurun_out/prof_pairbb_6.4_n256 -f python tools/case_single.py 6.4 256 f32 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:dmma -s 2 -c 1 -o gpurun_out/prof_dmma_1.3_n256 -f python tools/case_single.py 1.3 256 f64 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o gpurun_out/prof_small32_f32 -f python tools/small_single.py 32 1000000 f32 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o gpurun_out/prof_small32_f64 -f python tools/small_single.py 32 1000000 f64 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep_f32.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
ls -la gpurun_out
