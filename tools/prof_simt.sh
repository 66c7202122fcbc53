O=gpurun_out/s4h; mkdir -p $O
IALS_TC=0 timeout 300 bash tools/all_configs.sh mid sw-b16 > $O/all_tc0.txt 2>&1
IALS_TC=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_light -s 6 -c 1 -o $O/ncu_light32 python bench.py --config mid --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_light32.log 2>&1
python tools/ncu_summary.py $O/ncu_light32.ncu-rep $O/ncu_light32.txt > /dev/null 2>&1
python tools/ncu_stalls.py $O/ncu_light32.ncu-rep 30 > $O/ncu_light32_stalls.txt 2>&1
rm -f $O/ncu_light32.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_light -s 6 -c 1 -o $O/ncu_light16 python bench.py --config sw-b16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_light16.log 2>&1
python tools/ncu_summary.py $O/ncu_light16.ncu-rep $O/ncu_light16.txt > /dev/null 2>&1
python tools/ncu_stalls.py $O/ncu_light16.ncu-rep 30 > $O/ncu_light16_stalls.txt 2>&1
rm -f $O/ncu_light16.ncu-rep
