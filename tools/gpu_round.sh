#!/bin/bash
# One gpurun call: GPU tests, default bench line, all-config epoch times, the ncu launch
# list of the bench command and one `ncu --set full` capture of the top kernels.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG [skip-tests]'
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 600 bash tools/all_configs.sh > $O/all_configs.txt 2>&1
# launch list of one bench epoch (cold, serialised; share of step only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > $O/ncu_launch.log 2>&1
# full capture of one launch of each dominant kernel (after a warm epoch)
for K in k_sweep_tc4 k_pass_cache k_heavy_partial_tc4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o $O/ncu_$K python tools/profile_pass.py --config L1 > $O/ncu_$K.log 2>&1
done
echo done > $O/DONE
