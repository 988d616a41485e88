#!/bin/bash
mkdir -p gpurun_out
for t in 3 1; do
  LSRN_SKETCH_TILE=$t timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/kr.jsonl 2>&1 || echo "tile $t FAILED" >> gpurun_out/kr.jsonl
done
LSRN_SKETCH_TILE=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" >> gpurun_out/kr.jsonl 2>&1
