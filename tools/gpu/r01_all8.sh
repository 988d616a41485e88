#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py -q -x > gpurun_out/all8.log 2>&1; echo "tests rc=$?" >> gpurun_out/all8.log
timeout 600 python bench.py --config t4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 >> gpurun_out/all8.log 2>&1
LSRN_CSR_ROWDOT_ALL2=1 timeout 600 python bench.py --config t4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 >> gpurun_out/all8.log 2>&1
