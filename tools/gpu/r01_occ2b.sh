#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/occ2b.jsonl 2>&1
LSRN_ROWPASS_OCC=1 timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/occ2b.jsonl 2>&1
timeout 300 python tools/diag/rowpass_tune.py c2 >> gpurun_out/occ2b.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py -x -q >> gpurun_out/occ2b.jsonl 2>&1
