#!/bin/bash
# epoch time of every bench config (no CPU baseline / e2e), one JSON summary line each
for c in ${@:-tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 L1 L2}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'ms/epoch', d['ms_per_step'], 'phases', d['phases_ms'], 'roof', d['roofline']['bound'], d['roofline']['frac'], 'epoch_frac', d['roofline']['epoch_frac_of_roofline'])" || echo "$c failed"
done
