#!/bin/bash
mkdir -p gpurun_out
for sp in 0 2 4 8 13 16; do
  if [ $sp = 0 ]; then timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsplit.jsonl 2>&1;
  else LSRN_SKETCH_NSPLIT=$sp timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsplit.jsonl 2>&1; fi
done
