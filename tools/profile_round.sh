#!/bin/bash
# ncu captures of the dominant kernels at the bench configurations + launch
# lists.  Reports stay in /tmp/prof on the box (large); the counter summaries
# land in gpurun_out/ (copied to profiles/ afterwards).
mkdir -p gpurun_out /tmp/prof
TAG=${TAG:-r02}
NCU="ncu --set full --clock-control none --import-source on"
P=/tmp/prof
timeout 300 $NCU -k regex:dmma_gemm -s 2 -c 1 -o $P/dmma_1.3_n256 -f python tools/case_single.py 1.3 256 f64 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:dmma_gemm -s 2 -c 1 -o $P/dmma_bb_6.4_n256 -f python tools/case_single.py 6.4 256 f64 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o $P/group_plain_n256 -f python tools/group_single.py plain 256 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o $P/group_bb_n256 -f python tools/group_single.py bb 256 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o $P/pair_1.3_n256 -f python tools/case_single.py 1.3 256 f32 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o $P/small32_f32 -f python tools/small_single.py 32 1000000 f32 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o $P/small32_f64 -f python tools/small_single.py 32 1000000 f64 > /dev/null 2>&1
timeout 300 $NCU -k regex:small_mma -s 1 -c 1 -o $P/small64_f32 -f python tools/small_single.py 64 1000000 f32 > /dev/null 2>&1
timeout 300 $NCU -k regex:dmma_gemm -s 1 -c 1 -o $P/order4_f64 -f python bench.py --config order4 --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
# HOOI iteration kernels (graph nodes of the timed run)
timeout 600 $NCU -k regex:"pair_tma|ritz|gapply" --launch-skip 200 -c 12 -o $P/hooi_iter -f python bench.py --config hooi --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
NCU_TRAFFIC_JSON=gpurun_out/ncu_traffic.json python tools/ncu_summary.py gpurun_out/${TAG}_ncu_summary.md \
  $P/dmma_1.3_n256.ncu-rep:tc_dmma_f64/n256/f64 \
  $P/dmma_bb_6.4_n256.ncu-rep:tc_dmma_f64_bb/n256/f64 \
  $P/group_plain_n256.ncu-rep:tc_tf32x3_pair_group/n256/f32 \
  $P/group_bb_n256.ncu-rep:tc_tf32x3_pair_group_bb/n256/f32 \
  $P/pair_1.3_n256.ncu-rep:tc_tf32x3_pair_tma/n256/f32 \
  $P/small32_f32.ncu-rep:small32_mma_f32/n32/f32 \
  $P/small32_f64.ncu-rep:small_batched_dmma_f64/n32/f64 \
  $P/small64_f32.ncu-rep:small64_mma_f32/n64/f32 \
  $P/order4_f64.ncu-rep:tc_dmma_f64/n128/f64
ncu -i $P/hooi_iter.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/${TAG}_ncu_hooi_iter.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_sweep_f64.csv python bench.py --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_hooi_f32.csv python bench.py --config hooi --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out | tail -5
