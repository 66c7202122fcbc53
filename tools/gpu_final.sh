#!/bin/bash
# Re-measure the bench lines and the GPU suite with the final library (the ncu captures of
# tools/gpu_round2b.sh stay: the kernels they profile changed only in the Woodbury tiles).
#   gpurun --timeout 3000 -- 'bash tools/gpu_final.sh TAG'
TAG=${1:-r02c}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 900 python bench.py --config msd --steps 3 --warmup 2 > $O/bench_msd.json 2> $O/bench_msd.err
timeout 600 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded_L1.json 2> $O/bench_sharded_L1.err
timeout 1500 bash tools/all_configs.sh tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 ials-d512 d64 d512 L1 L2 msd > $O/all_configs.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file $O/launches_L1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_L1.csv > $O/launches_L1_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_wb -s 20 -c 1 \
  -o $O/ncu_k_sweep_wb python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k_sweep_wb.log 2>&1
python tools/ncu_summary.py $O/ncu_k_sweep_wb.ncu-rep $O/ncu_k_sweep_wb.txt > /dev/null 2>&1
python tools/ncu_stalls.py $O/ncu_k_sweep_wb.ncu-rep 30 > $O/ncu_k_sweep_wb_stalls.txt 2>&1
rm -f $O/ncu_k_sweep_wb.ncu-rep
echo done > $O/DONE
