#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowpass.py -q -x -k "wide or rowpass" > gpurun_out/rp7.log 2>&1; echo "rc=$?" >> gpurun_out/rp7.log
timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/rp7.log 2>&1
