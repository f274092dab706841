mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; tail -3 gpurun_out/g1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; tail -2 gpurun_out/g1_smoke.log
timeout 300 python bench.py --config hooi > gpurun_out/g1_hooi_f32.json 2>&1
timeout 300 python bench.py --config hooi --dtype f64 > gpurun_out/g1_hooi_f64.json 2>&1
timeout 300 python bench.py --dtype f64 > gpurun_out/g1_sweep_f64.json 2>&1
