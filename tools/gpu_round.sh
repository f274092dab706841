#!/bin/bash
# One GPU session: tests, bench lines for every config, launch list and ncu captures.
set -x
mkdir -p gpurun_out
timeout 1000 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_sweep_f32.json 2> gpurun_out/bench_sweep_f32.err
timeout 300 python bench.py --dtype f64 --no-e2e > gpurun_out/bench_sweep_f64.json 2> gpurun_out/bench_sweep_f64.err
timeout 300 python bench.py --n 512 --no-e2e --no-cpu --steps 5 > gpurun_out/bench_sweep_f32_n512.json 2>&1
timeout 300 python bench.py --n 128 --no-e2e --no-cpu > gpurun_out/bench_sweep_f32_n128.json 2>&1
timeout 300 python bench.py --n 64 --no-e2e --no-cpu > gpurun_out/bench_sweep_f32_n64.json 2>&1
timeout 300 python bench.py --n 64 --dtype f64 --no-e2e --no-cpu > gpurun_out/bench_sweep_f64_n64.json 2>&1
timeout 300 python bench.py --n 512 --dtype f64 --no-e2e --no-cpu --steps 3 > gpurun_out/bench_sweep_f64_n512.json 2>&1
timeout 300 python bench.py --n 1024 --no-e2e --no-cpu --steps 3 > gpurun_out/bench_sweep_f32_n1024.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1
for dt in f32 f64; do
  timeout 300 python bench.py --config small --dtype $dt > gpurun_out/bench_small_$dt.json 2>&1
  timeout 300 python bench.py --config order4 --dtype $dt > gpurun_out/bench_order4_$dt.json 2>&1
done
timeout 400 python bench.py --config hooi > gpurun_out/bench_hooi_f32.json 2>&1
timeout 400 python bench.py --config hooi --dtype f64 > gpurun_out/bench_hooi_f64.json 2>&1
timeout 300 python bench.py --config conventional --no-e2e > gpurun_out/bench_conventional_f32.json 2>&1
bash tools/profile_round.sh
ls -la gpurun_out
