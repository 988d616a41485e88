#!/bin/bash
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_multirank_host.py -m gpu -x -q -p no:cacheprovider -k full_c5 --durations=3 > gpurun_out/r02/pytest_full2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_full2.log; tail -8 gpurun_out/r02/pytest_full2.log
