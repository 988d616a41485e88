#!/bin/bash
mkdir -p gpurun_out
for tile in 0 1 2; do
  for cl in 1 2; do
    LSRN_SKETCH_TILE=$tile LSRN_SKETCH_MAXCL=$cl timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/tile.jsonl 2>&1 || echo "tile=$tile cl=$cl FAILED" >> gpurun_out/tile.jsonl
  done
done
LSRN_SKETCH_TILE=1 LSRN_SKETCH_DIAG=1 timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/tile.jsonl 2>&1
LSRN_SKETCH_TILE=1 timeout 120 python tools/diag/sketch_tune.py 1000000 10000 >> gpurun_out/tile.jsonl 2>&1
for tile in 1 2; do
  LSRN_SKETCH_TILE=$tile timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch" >> gpurun_out/tile.jsonl 2>&1
done
