#!/bin/bash
# round-2 re-entry validation: the full gpu suite, smoke, the default and
# per-config bench lines, 2 ranks sharing one GPU, the reference suite on b200
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > gpurun_out/g3_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/g3_pytest.log 2>&1; tail -25 gpurun_out/g3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g3_smoke.log 2>&1; tail -2 gpurun_out/g3_smoke.log
timeout 400 python bench.py > gpurun_out/g3_bench_default.json 2> gpurun_out/g3_bench_default.err
timeout 300 python bench.py --impl reference > gpurun_out/g3_bench_reference.json 2> gpurun_out/g3_bench_reference.err
for c in c1 small order4 hooi; do
  timeout 400 python bench.py --config $c > gpurun_out/g3_bench_$c.json 2> gpurun_out/g3_bench_$c.err
done
SBT_SHARE_GPU=1 timeout 300 python bench.py --gpus 2 --config c1 --no-e2e --steps 3 > gpurun_out/g3_bench_c1_2ranks.json 2> gpurun_out/g3_bench_c1_2ranks.err
timeout 900 bash tools/run_ref_suite.sh > gpurun_out/g3_ref_suite.log 2>&1; tail -5 gpurun_out/g3_ref_suite.log
tail -n1 gpurun_out/g3_bench_*.json
