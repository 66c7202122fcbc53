#!/bin/bash
# ncu launch lists (gpu__time_duration.sum, cold, serialised) of one bench epoch per config:
#   gpurun --timeout 1500 -- 'bash tools/launches_cfg.sh TAG cfg1 cfg2 ...'
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for c in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
  python tools/launch_summary.py $O/launches_$c.csv > $O/launches_${c}_summary.txt 2>&1
done
