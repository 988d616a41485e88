#!/bin/bash
# producer-warp variants of the dense sketch (NPW = 4 interleaved pairs vs 8)
mkdir -p gpurun_out
for npw in 4 8; do
  for cl in 2 4; do
    LSRN_SKETCH_NPW=$npw LSRN_SKETCH_MAXCL=$cl timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/npw.jsonl 2>&1 || echo "npw=$npw cl=$cl FAILED rc=$?" >> gpurun_out/npw.jsonl
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch or gaussian" >> gpurun_out/npw.jsonl 2>&1
tail -3 gpurun_out/npw.jsonl
