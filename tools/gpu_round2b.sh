#!/bin/bash
# Round-2 final measurement record (one gpurun call):
#   gpurun --timeout 4500 -- 'bash tools/gpu_round2b.sh TAG'
# the GPU suite (product library, then the bounds-checked build on the parity files),
# bench lines (L1 default, mid, msd, sharded L1, the reference arm), every config's epoch
# time, the ncu launch list and DRAM traffic of the L1 bench epoch, and one
# `ncu --set full` capture per dominant kernel (each command first ran clean without ncu).
TAG=${1:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
IALS_LIB=checked timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_eval.py -m gpu -q > $O/pytest_checked.log 2>&1; echo "rc=$?" >> $O/pytest_checked.log
timeout 600 python bench.py > $O/bench_L1.json 2> $O/bench_L1.err
timeout 600 python bench.py --config mid > $O/bench_mid.json 2> $O/bench_mid.err
timeout 900 python bench.py --config msd --steps 3 --warmup 2 > $O/bench_msd.json 2> $O/bench_msd.err
timeout 600 python bench.py --sharded --no-cpu-baseline > $O/bench_sharded_L1.json 2> $O/bench_sharded_L1.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1500 bash tools/all_configs.sh tiny mid sw-b1 sw-b16 sw-b64 sw-b128 sw-b256 ials-d512 d64 d512 L1 L2 msd > $O/all_configs.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file $O/launches_L1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_L1.csv > $O/launches_L1_summary.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -c 600 --csv --log-file $O/traffic_L1_ncu_metrics.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_traffic.log 2>&1
summarise() {   # the report is summarised on the box and dropped (gpurun_out <= 64 MiB)
  python tools/ncu_summary.py $O/ncu_$1.ncu-rep $O/ncu_$1.txt > /dev/null 2>&1
  python tools/ncu_stalls.py $O/ncu_$1.ncu-rep 30 > $O/ncu_$1_stalls.txt 2>&1
  rm -f $O/ncu_$1.ncu-rep
}
for K in k_sweep_tc4 k_sweep_wb k_pass_cache_flat k_heavy_partial_tc4 k_pred_vec; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 \
    -o $O/ncu_$K python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_$K.log 2>&1
  summarise $K
done
# the GEMMs of the timed epoch's block 0 (72 launches per epoch: the diagonal blocks, then per
# block H slab, (slab Q)^T, user projection, F~, W Q, back-rotation, W slab, item projection,
# the next epoch's diagonal block): launch 75 = the user projection (1068 CTAs), 79 = the W slab
for N in 75 79; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm3_tf32 -s $N -c 1 \
    -o $O/ncu_k_gemm3_tf32_$N python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k_gemm3_tf32_$N.log 2>&1
  summarise k_gemm3_tf32_$N
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pk -s 4 -c 1 \
  -o $O/ncu_k_sweep_pk python bench.py --config mid --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_k_sweep_pk.log 2>&1
summarise k_sweep_pk
echo done > $O/DONE
