#!/bin/bash
O=gpurun_out/exp2; mkdir -p $O
IALS_DEFER_CACHE=0 timeout 300 bash tools/all_configs.sh L1 msd mid > $O/nodefer.txt 2>&1
timeout 300 bash tools/all_configs.sh L1 msd mid > $O/defer.txt 2>&1
