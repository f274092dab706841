#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/g21_pytest.log 2>&1; tail -15 gpurun_out/g21_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g21_smoke.log 2>&1; tail -2 gpurun_out/g21_smoke.log
