#!/bin/bash
mkdir -p gpurun_out
for pf in 0 1; do
  LSRN_SKETCH_PFIRST=$pf timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/pf.jsonl 2>&1 || echo "pf $pf FAILED" >> gpurun_out/pf.jsonl
done
LSRN_SKETCH_PFIRST=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" >> gpurun_out/pf.jsonl 2>&1
