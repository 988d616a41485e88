#!/bin/bash
mkdir -p gpurun_out
LSRN_FULLSIZE=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize.log
tail -3 gpurun_out/fullsize.log
