#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsplit2.jsonl 2>&1
for sp in 5 7 10 12 13; do
  LSRN_SKETCH_NSPLIT=$sp timeout 120 python tools/diag/sketch_tune.py 100000 2000 >> gpurun_out/nsplit2.jsonl 2>&1
done
timeout 120 python tools/diag/sketch_tune.py 200000 2000 >> gpurun_out/nsplit2.jsonl 2>&1
LSRN_SKETCH_NSPLIT=13 timeout 120 python tools/diag/sketch_tune.py 200000 2000 >> gpurun_out/nsplit2.jsonl 2>&1
