#!/bin/bash
O=gpurun_out/exp1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_golden.py -x -q -k "rot or woodbury or golden or tensor_core or sharded or dropin" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 bash tools/all_configs.sh L1 sw-b128 > $O/all.txt 2>&1
IALS_HEAVY=2048 timeout 300 bash tools/all_configs.sh L1 > $O/heavy2048.txt 2>&1
IALS_HEAVY=1024 IALS_SLICE=1024 timeout 300 bash tools/all_configs.sh L1 > $O/heavy1024.txt 2>&1
IALS_HEAVY=2048 IALS_SLICE=1024 timeout 300 bash tools/all_configs.sh L1 > $O/heavy2048_s1024.txt 2>&1
for c in tiny sw-b1 sw-b16; do timeout 300 python tools/graph_check.py $c > $O/graph_$c.txt 2>&1; done
