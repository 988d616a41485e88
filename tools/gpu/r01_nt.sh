#!/bin/bash
mkdir -p gpurun_out
for nt in 512 256; do
  LSRN_ROWPASS_NT=$nt timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/nt.jsonl 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q >> gpurun_out/nt.jsonl 2>&1
