#!/bin/bash
# One GPU session: the gpu test suite, smoke, a bench line for every config
# (default = the fp64 36-case sweep headline), the reference arm.
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${TAG:-r02}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${TAG}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
B() { out=$1; shift; timeout 400 python bench.py "$@" > gpurun_out/${TAG}_bench_$out.json 2> gpurun_out/${TAG}_bench_$out.err; tail -c 300 gpurun_out/${TAG}_bench_$out.json | head -c 0; }
B sweep_f64
B sweep_f32 --dtype f32
B sweep_f64_n128 --dtype f64 --n 128 --no-e2e --no-cpu
B sweep_f64_n512 --dtype f64 --n 512 --no-e2e --no-cpu --steps 3
B sweep_f32_n512 --dtype f32 --n 512 --no-e2e --no-cpu --steps 5
B sweep_f32_n1024 --dtype f32 --n 1024 --no-e2e --no-cpu --steps 3
B c1 --config c1
B c1_f32 --config c1 --dtype f32 --no-cpu
B small_f32 --config small --dtype f32
B small_f64 --config small --dtype f64
B order4_f64 --config order4 --dtype f64
B order4_f32 --config order4 --dtype f32
B hooi_f32 --config hooi
B hooi_f64 --config hooi --dtype f64 --no-e2e
B conventional_f64 --config conventional --dtype f64 --no-e2e
B reference --impl reference
timeout 900 bash tools/run_ref_suite.sh > gpurun_out/${TAG}_ref_suite.log 2>&1; tail -1 gpurun_out/${TAG}_ref_suite.log
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), d.get('unit'), 'frac', (d.get('roofline') or {}).get('frac'), 'ms', d.get('ms_per_step'))" 2>&1 | tail -1)"; done
