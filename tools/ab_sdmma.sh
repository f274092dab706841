#!/bin/bash
export PYTHONDONTWRITEBYTECODE=1
for lib in libsbt200 libsbt200_sd1; do
  SBT_LIB=$PWD/paper_1606_05696_b200/lib/$lib.so timeout 300 python bench.py --config small --dtype f64 --no-e2e --no-cpu > gpurun_out/ab_sd_$lib.json 2>&1
  python - $lib <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_sd_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], [(e["n"], e["kernel"], e["frac_of_measured_hbm"], e["gflops"]) for e in d["sweep"]])
PY
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "small or batched" 2>&1 | tail -1
