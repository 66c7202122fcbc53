#!/bin/bash
# per-line instruction distribution of the user-pass and item-pass k_sweep_tc4 launches at L1
O=gpurun_out/tc4_lines; mkdir -p $O
R="ials_sweep_tc4.cuh:init:81-107 ials_sweep_tc4.cuh:meta+gather:108-175 ials_sweep_tc4.cuh:accumulate:176-318 ials_sweep_tc4.cuh:factor:319-513 ials_sweep_tc4.cuh:block_inverses:514-539 ials_sweep_tc4.cuh:backward:540-581 ials_sweep_tc4.cuh:kernel_body:582-751"
for S in 16 17; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_tc4 -s $S -c 1 \
    -o $O/tc4_$S python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/tc4_$S.log 2>&1
  python tools/ncu_lines_inst.py $O/tc4_$S.ncu-rep 70 $R > $O/tc4_${S}_inst.txt 2>&1
  python tools/ncu_summary.py $O/tc4_$S.ncu-rep $O/tc4_${S}_sum.txt > /dev/null 2>&1
  rm -f $O/tc4_$S.ncu-rep
done
