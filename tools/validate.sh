#!/bin/bash
# Focused GPU validation after a kernel change (run under gpurun):
#   bash tools/validate.sh f64 | hooi | small | ranks
# f64:   fp64 parity subset + the fp64 bench lines (sweep, C1, 4th order, HOOI)
# hooi:  HOOI / factor-update parity (incl. the 512^3 rank-32 oracle test) + HOOI bench
# small: small-matrix parity + the batched sweep (mma.sync vs FFMA: SBT_SMALL_MMA=0)
# ranks: two ranks sharing the GPU (gloo): sharded HOOI and batched shards end to end
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out
case "$1" in
f64)
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_conventional.py -q -x -k "f64 or dmma or 36 or c1 or hooi or float64" 2>&1 | tail -1
  for c in "sweep_f64" "c1 --config c1" "order4_f64 --config order4 --dtype f64" "hooi_f64 --config hooi --dtype f64 --no-e2e"; do
    set -- $c; name=$1; shift
    timeout 400 python bench.py "$@" > gpurun_out/val_$name.json 2>&1
    echo "$name: $(grep -o '"value": [0-9.]*' gpurun_out/val_$name.json | head -1) $(grep -o '"frac": [0-9.]*' gpurun_out/val_$name.json | head -1)"
  done ;;
hooi)
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "hooi or factor or acc64 or narrow or long" 2>&1 | tail -1
  timeout 400 python bench.py --config hooi --no-e2e --no-cpu > gpurun_out/val_hooi.json 2>&1
  grep -o '"ms_per_iteration": [0-9.]*\|"fit_history": \[[0-9.]*\|"frac": [0-9.]*' gpurun_out/val_hooi.json | head -3 ;;
small)
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -k "small or batched" 2>&1 | tail -1
  for dt in f32 f64; do
    timeout 300 python bench.py --config small --dtype $dt --no-e2e --no-cpu > gpurun_out/val_small_$dt.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/val_small_$dt.json').read().strip().splitlines()[-1]); print('$dt', [(e['n'], e['kernel'], e['frac_of_measured_hbm']) for e in d['sweep']])"
  done ;;
ranks)
  SBT_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config hooi --no-cpu --steps 2 > gpurun_out/val_ranks_hooi.json 2> gpurun_out/val_ranks_hooi.err; tail -c 400 gpurun_out/val_ranks_hooi.json
  SBT_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config small --no-e2e --no-cpu --steps 3 > gpurun_out/val_ranks_small.json 2> gpurun_out/val_ranks_small.err; tail -c 300 gpurun_out/val_ranks_small.json ;;
*) echo "usage: $0 f64|hooi|small|ranks"; exit 2 ;;
esac
