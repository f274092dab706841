#!/bin/bash
# A/B: CTA-pair tile width 256 vs 128 for the fp32 sweep (grouped and single calls)
for b in 0 128; do
  SBT_TC_BNT=$b timeout 300 python bench.py --dtype f32 --no-e2e --no-cpu --steps 5 > gpurun_out/ab_bnt$b.json 2>&1
  python - $b <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_bnt{sys.argv[1]}.json").read().strip().splitlines()[-1])
pc = d["per_case"]
single = sum(v["ms"] for v in pc.values())
print("BNT cap", sys.argv[1], "value", d["value"], d["group_launches"], "sum of single calls ms", round(single, 3),
      "single-call TF/s", round(36 * 2 * 256 ** 4 / single / 1e9, 1))
PY
done
