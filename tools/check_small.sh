#!/bin/bash
# fp32 small batched: mma.sync kernels (n = 32 / 64) vs the FFMA kernels
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -k "small or batched" 2>&1 | tail -1
for v in 1 0; do
  SBT_SMALL_MMA=$v timeout 300 python bench.py --config small --dtype f32 --no-e2e --no-cpu > gpurun_out/chk_small_mma$v.json 2>&1
  python - $v <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/chk_small_mma{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("mma", sys.argv[1], [(e["n"], e["kernel"], e["frac_of_measured_hbm"]) for e in d["sweep"]])
PY
done
