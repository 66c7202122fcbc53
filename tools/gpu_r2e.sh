#!/bin/bash
# Session-5 record of round 2 (after the warp-level narrow-width kernels): the GPU suite with
# the product library and with the bounds-checked build, the bench lines, the reference arm,
# every config, launch lists (L1, mid) and one ncu capture per new kernel.
#   gpurun --timeout 3400 -- 'bash tools/gpu_r2e.sh TAG'
TAG=${1:-r02e}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded_L1.json 2> $O/bench_sharded_L1.err
timeout 1500 bash tools/all_configs.sh tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 d64 d512 L1 L2 msd > $O/all_configs.txt 2>&1
IALS_LIB=checked timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_eval.py -q > $O/pytest_checked.log 2>&1; echo "rc=$?" >> $O/pytest_checked.log
for c in L1 mid sw-b16; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1
  python tools/launch_summary.py $O/launches_$c.csv > $O/launches_${c}_summary.txt 2>&1
done
cap() {  # kernel regex, config, skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $3 -c 1 \
    -o $O/ncu_$1 python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_$1.log 2>&1
  python tools/ncu_summary.py $O/ncu_$1.ncu-rep $O/ncu_$1.txt > /dev/null 2>&1
  python tools/ncu_stalls.py $O/ncu_$1.ncu-rep 30 > $O/ncu_$1_stalls.txt 2>&1
  rm -f $O/ncu_$1.ncu-rep
}
cap k_sweep_w32m mid 4
cap k_heavy_partial_wm mid 3
cap k_sweep_w16m sw-b16 4
cap k_b1_cache_flat sw-b1 3
echo done > $O/DONE
