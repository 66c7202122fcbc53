#!/bin/bash
O=gpurun_out/exp3; mkdir -p $O
timeout 300 bash tools/all_configs.sh L1 mid sw-b64 sw-b128 > $O/all.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_golden.py tests/test_gpu_fullscale.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 bash tools/all_configs.sh msd L2 d64 >> $O/all.txt 2>&1
