#!/bin/bash
# Round-end evidence for profiles/: bench lines (configs 1-5, reference arm),
# the config-4 launch list, ncu --set full captures of the epoch kernel
# (configs 2, 3, 4) and per-phase timelines (configs 2 and 4).  Run from the
# repo root on the GPU box:
#   bash tools/round_profiles.sh TAG     -> gpurun_out/TAG_*
set -x
T=${1:-r02f}
O=gpurun_out
for c in 4 3 2 1 5; do
  python bench.py --config $c > $O/${T}_bench_cfg$c.json 2> $O/${T}_bench_cfg$c.err
done
python bench.py --impl reference > $O/${T}_bench_cfg4_reference.json 2> $O/${T}_ref.err
python tools/phase_timeline.py --config 2 > $O/${T}_timeline_cfg2.txt 2>&1
python tools/phase_timeline.py --config 4 --batched > $O/${T}_timeline_cfg4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 7000 --csv \
    --log-file $O/${T}_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
for c in 4 3 2; do
  ncu --set full --clock-control none --import-source on -k regex:epoch_kernel -s 6 -c 1 \
      -o $O/${T}_cfg$c python bench.py --config $c --steps 4 --warmup 3 --no-cpu > $O/${T}_ncu_cfg$c.log 2>&1
done
ls -la $O/${T}_*
