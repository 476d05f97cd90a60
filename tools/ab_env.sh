#!/bin/bash
# Same-box A/B of an environment switch: tools/ab_env.sh REPS CONFIG VAR v1 v2 ...
REPS=$1; CFG=$2; VAR=$3; shift 3
for i in $(seq $REPS); do
  for v in "$@"; do
    env $VAR=$v python bench.py --no-cpu --steps 30 --config $CFG > gpurun_out/abe_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/abe_$v.json'));print('$VAR=$v', round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4))"
  done
done
