#!/bin/bash
mkdir -p gpurun_out
for cfg in "1 256" "1 512" "0 256"; do
  set -- $cfg
  LSRN_ROWPASS_XFLOW=$1 LSRN_ROWPASS_NT=$2 timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/xflow.jsonl 2>&1 || echo "FAILED $cfg" >> gpurun_out/xflow.jsonl
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q >> gpurun_out/xflow.jsonl 2>&1
