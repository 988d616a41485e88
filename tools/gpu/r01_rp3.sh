#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowpass.py tests/test_gpu_parity.py -q -x > gpurun_out/rp3.log 2>&1; echo "tests rc=$?" >> gpurun_out/rp3.log
for shape in "20000 20000" "125000 10000" "100000 2000" "20000 15000" "20000 30000"; do
  timeout 120 python tools/diag/rowpass_shape.py $shape >> gpurun_out/rp3.log 2>&1
done
