#!/bin/bash
# Round-2 measurement record (one gpurun call):
#   gpurun --timeout 3000 -- 'bash tools/gpu_round2.sh TAG'
# bench lines (L1 default, mid = configs[1], msd = configs[4], the reference arm),
# the ncu launch list and DRAM traffic of the L1 bench epoch, and one
# `ncu --set full` capture per dominant kernel (each command first ran clean).
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 900 python bench.py --config msd --steps 3 --warmup 2 > $O/bench_msd.json 2> $O/bench_msd.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/launches_L1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -c 400 --csv --log-file $O/traffic_L1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_traffic.log 2>&1
summarise() {   # the report is summarised on the box and dropped (gpurun_out <= 64 MiB)
  python tools/ncu_summary.py $O/ncu_$1.ncu-rep $O/ncu_$1.txt > /dev/null 2>&1
  python tools/ncu_stalls.py $O/ncu_$1.ncu-rep 30 > $O/ncu_$1_stalls.txt 2>&1
  rm -f $O/ncu_$1.ncu-rep
}
for K in k_sweep_tc4 k_sweep_wb k_gemm3_tf32 k_pass_cache_flat k_heavy_partial_tc4 k_sym_eig k_pred_vec; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
    -o $O/ncu_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_$K.log 2>&1
  summarise $K
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pk -s 4 -c 1 \
  -o $O/ncu_k_sweep_pk python bench.py --config mid --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k_sweep_pk.log 2>&1
summarise k_sweep_pk
echo done > $O/DONE
