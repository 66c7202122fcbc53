#!/bin/bash
# Session-5 record of round 2: the GPU suite, the bench lines, every config, the mid launch
# list and one ncu capture of the warp-per-row sweep (k_sweep_w32), with the current library.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2d.sh TAG'
TAG=${1:-r02d}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 1500 bash tools/all_configs.sh tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 d64 d512 L1 L2 > $O/all_configs.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file $O/launches_mid.csv python bench.py --config mid --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_mid.log 2>&1
python tools/launch_summary.py $O/launches_mid.csv > $O/launches_mid_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_w32 -s 4 -c 1 \
  -o $O/ncu_k_sweep_w32 python bench.py --config mid --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k_sweep_w32.log 2>&1
python tools/ncu_summary.py $O/ncu_k_sweep_w32.ncu-rep $O/ncu_k_sweep_w32.txt > /dev/null 2>&1
python tools/ncu_stalls.py $O/ncu_k_sweep_w32.ncu-rep 30 > $O/ncu_k_sweep_w32_stalls.txt 2>&1
rm -f $O/ncu_k_sweep_w32.ncu-rep
echo done > $O/DONE
