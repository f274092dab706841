#!/bin/bash
# A/B an environment switch on one bench config, repeated: ab_env.sh "<bench args>" VAR val1 val2 [reps]
args=$1; var=$2; v1=$3; v2=$4; reps=${5:-2}
for rep in $(seq 1 $reps); do for v in $v1 $v2; do
  env $var=$v timeout 400 python bench.py $args > gpurun_out/ab_env.json 2>&1
  echo "rep$rep $var=$v $(grep -o '"value": [0-9.]*' gpurun_out/ab_env.json | head -1) $(grep -o '"group_launches": {[^}]*}[^}]*}' gpurun_out/ab_env.json | head -c 240)"
done; done
