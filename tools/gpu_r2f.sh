#!/bin/bash
# Final re-measurement of the session (after the cancellation guards of the warp-level MMA
# sweeps and the 64-wide slice kernel): GPU suite with both builds, bench lines, every config.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2f.sh TAG'
TAG=${1:-r02f}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 1500 bash tools/all_configs.sh tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 d64 d512 L1 L2 msd > $O/all_configs.txt 2>&1
IALS_LIB=checked timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_eval.py -q > $O/pytest_checked.log 2>&1; echo "rc=$?" >> $O/pytest_checked.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for c in mid sw-b16 sw-b64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1
  python tools/launch_summary.py $O/launches_$c.csv > $O/launches_${c}_summary.txt 2>&1
done
echo done > $O/DONE
