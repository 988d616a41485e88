#!/bin/bash
mkdir -p gpurun_out
LSRN_ROWPASS_WIDE1=1 timeout 120 python tools/diag/rowpass_shape.py 125000 10000 >> gpurun_out/rp6.log 2>&1 || echo "FAILED wide1" >> gpurun_out/rp6.log
timeout 120 python tools/diag/rowpass_shape.py 125000 10000 >> gpurun_out/rp6.log 2>&1
LSRN_ROWPASS_WIDE1=1 timeout 120 python tools/diag/rowpass_shape.py 20000 10000 >> gpurun_out/rp6.log 2>&1 || echo "FAILED wide1 b" >> gpurun_out/rp6.log
timeout 120 python tools/diag/rowpass_shape.py 20000 10000 >> gpurun_out/rp6.log 2>&1
LSRN_ROWPASS_WIDE1=1 timeout 300 python -m pytest tests/test_gpu_rowpass.py -q -x >> gpurun_out/rp6.log 2>&1
