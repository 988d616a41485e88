#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py -x -q > gpurun_out/csrhl.log 2>&1; echo "tests rc=$?" >> gpurun_out/csrhl.log
timeout 300 python tools/diag/csr_longpass.py 2000000 4000 >> gpurun_out/csrhl.log 2>&1
LSRN_CSR_ROWDOT_V1=1 timeout 300 python tools/diag/csr_longpass.py 2000000 4000 >> gpurun_out/csrhl.log 2>&1
