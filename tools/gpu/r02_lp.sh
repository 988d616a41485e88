#!/bin/bash
mkdir -p gpurun_out/r02
timeout 400 python -m pytest tests/test_gpu_csr.py tests/test_gpu_nccl1.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02/pytest_lp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_lp.log; tail -3 gpurun_out/r02/pytest_lp.log
timeout 300 python tools/diag/csr_longpass_variants.py t4 -1 2>&1 | tail -3
