#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowpass.py -q -x > gpurun_out/rp.log 2>&1; echo "tests rc=$?" >> gpurun_out/rp.log
for shape in "20000 20000" "125000 10000" "100000 2000"; do
  timeout 120 python tools/diag/rowpass_shape.py $shape >> gpurun_out/rp.log 2>&1
done
for env in "LSRN_ROWPASS_OCC=1" "LSRN_ROWPASS_WIDE_SLICE=10000" "LSRN_ROWPASS_WIDE_SLICE=10000 LSRN_ROWPASS_OCC=1" "LSRN_ROWPASS_WIDE_SLICE=5000" "LSRN_ROWPASS_WIDE_SLICE=4096"; do
  env $env timeout 120 python tools/diag/rowpass_shape.py 20000 20000 >> gpurun_out/rp.log 2>&1 || echo "FAILED $env" >> gpurun_out/rp.log
done
