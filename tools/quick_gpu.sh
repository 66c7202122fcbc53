#!/bin/bash
# One gpurun call for kernel iteration: the narrow/packed parity tests and the
# epoch times of the given configs.
#   gpurun --timeout 1500 -- 'bash tools/quick_gpu.sh TAG "pytest -k expr" cfg1 cfg2 ...'
TAG=$1; shift
K=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -x -q -k "$K" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 900 bash tools/all_configs.sh "$@" > $O/all.txt 2>&1
