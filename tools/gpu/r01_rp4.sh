#!/bin/bash
mkdir -p gpurun_out
for shape in "20000 20000" "20000 16000"; do
  LSRN_ROWPASS_WIDE2=1 timeout 120 python tools/diag/rowpass_shape.py $shape >> gpurun_out/rp4.log 2>&1 || echo "FAILED wide2 $shape" >> gpurun_out/rp4.log
  timeout 120 python tools/diag/rowpass_shape.py $shape >> gpurun_out/rp4.log 2>&1
done
LSRN_ROWPASS_WIDE2=1 timeout 300 python -m pytest tests/test_gpu_rowpass.py -q -x >> gpurun_out/rp4.log 2>&1
