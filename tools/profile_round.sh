#!/bin/bash
# ncu captures of the dominant kernels at the bench configurations + launch list.
# Reports stay in /tmp/prof on the box (too large to bring back); the counter
# summaries land in gpurun_out/ (copied to profiles/ afterwards).
mkdir -p gpurun_out /tmp/prof
TAG=${TAG:-r01g}
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o /tmp/prof/pair_1.3_n256 -f python tools/case_single.py 1.3 256 f32 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o /tmp/prof/group_plain_n256 -f python tools/group_single.py plain 256 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o /tmp/prof/group_bb_n256 -f python tools/group_single.py bb 256 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 2 -c 1 -o /tmp/prof/pairbb_6.4_n256 -f python tools/case_single.py 6.4 256 f32 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:dmma -s 2 -c 1 -o /tmp/prof/dmma_1.3_n256 -f python tools/case_single.py 1.3 256 f64 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:dmma -s 2 -c 1 -o /tmp/prof/dmma_bb_6.4_n256 -f python tools/case_single.py 6.4 256 f64 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o /tmp/prof/small32_f32 -f python tools/small_single.py 32 1000000 f32 > /dev/null 2>&1
timeout 300 $NCU -k regex:small -s 1 -c 1 -o /tmp/prof/small32_f64 -f python tools/small_single.py 32 1000000 f64 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 1 -c 1 -o /tmp/prof/fold_order4 -f python bench.py --config order4 --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 $NCU -k regex:pair_tma -s 0 -c 1 -o /tmp/prof/hooi_narrow -f python tools/hooi_products.py > /dev/null 2>&1
timeout 300 $NCU -k regex:ritz -s 2 -c 1 -o /tmp/prof/ritz -f python tools/ritz_probe.py > /dev/null 2>&1
timeout 300 $NCU -k regex:skinny -s 3 -c 1 -o /tmp/prof/skinny -f python tools/skinny_probe.py > /dev/null 2>&1
NCU_TRAFFIC_JSON=gpurun_out/ncu_traffic.json python tools/ncu_summary.py gpurun_out/${TAG}_ncu_summary.md \
  /tmp/prof/hooi_narrow.ncu-rep:tc_tf32x3_pair_narrow/hooi512/f32 \
  /tmp/prof/ritz.ncu-rep:ritz_f64/hooi512/f64 \
  /tmp/prof/skinny.ncu-rep:skinny_dmma_f64/hooi512/f64 \
  /tmp/prof/pair_1.3_n256.ncu-rep:tc_tf32x3_pair_tma/n256/f32 \
  /tmp/prof/group_plain_n256.ncu-rep:tc_tf32x3_pair_group/n256/f32 \
  /tmp/prof/group_bb_n256.ncu-rep:tc_tf32x3_pair_group_bb/n256/f32 \
  /tmp/prof/pairbb_6.4_n256.ncu-rep:tc_tf32x3_pair_bb/n256/f32 \
  /tmp/prof/dmma_1.3_n256.ncu-rep:tc_dmma_f64/n256/f64 \
  /tmp/prof/dmma_bb_6.4_n256.ncu-rep:tc_dmma_f64_bb/n256/f64 \
  /tmp/prof/small32_f32.ncu-rep:small_batched_f32/n32/f32 \
  /tmp/prof/small32_f64.ncu-rep:small_batched_dmma_f64/n32/f64 \
  /tmp/prof/fold_order4.ncu-rep:tc_tf32x3_pair_fold/n128/f32
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sweep_f32.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hooi_f32.csv python bench.py --config hooi --steps 3 > /dev/null 2>&1
ls -la gpurun_out
