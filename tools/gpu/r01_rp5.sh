#!/bin/bash
mkdir -p gpurun_out
for env in "LSRN_ROWPASS_TR=2 LSRN_ROWPASS_OCC=1" "LSRN_ROWPASS_TR=2 LSRN_ROWPASS_OCC=1 LSRN_ROWPASS_BUDGET_KB=224" "LSRN_ROWPASS_TR=1"; do
  env $env timeout 120 python tools/diag/rowpass_shape.py 125000 10000 >> gpurun_out/rp5.log 2>&1 || echo "FAILED $env" >> gpurun_out/rp5.log
done
for env in "LSRN_ROWPASS_TR=2 LSRN_ROWPASS_OCC=2" "LSRN_ROWPASS_TR=2 LSRN_ROWPASS_OCC=1"; do
  env $env timeout 120 python tools/diag/rowpass_shape.py 100000 6000 >> gpurun_out/rp5.log 2>&1 || echo "FAILED $env" >> gpurun_out/rp5.log
done
timeout 120 python tools/diag/rowpass_shape.py 100000 6000 >> gpurun_out/rp5.log 2>&1
