#!/bin/bash
mkdir -p gpurun_out
for nsg in 4 6 8; do
  LSRN_SKETCH_NSG=$nsg timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsg.jsonl 2>&1 || echo "nsg=$nsg FAILED" >> gpurun_out/nsg.jsonl
done
LSRN_SKETCH_NSG=8 LSRN_SKETCH_MAXCL=4 timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsg.jsonl 2>&1
LSRN_SKETCH_NSG=8 LSRN_SKETCH_DIAG=1 timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsg.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch or gaussian" >> gpurun_out/nsg.jsonl 2>&1
