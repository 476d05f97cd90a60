#!/bin/bash
# Same-box A/B of library variants: tools/ab.sh REPS CONFIG variant...  ("base" = default build)
REPS=$1; CFG=$2; shift 2
for i in $(seq $REPS); do
  for v in "$@"; do
    if [ "$v" = base ]; then unset BCT_LIB; else export BCT_LIB=paper_1709_00953_b200/_lib/libblockct_cuda_$v.so; fi
    python bench.py --no-cpu --steps 30 --config $CFG > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4))"
  done
done
