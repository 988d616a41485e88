#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfg in "LSRN_SKETCH_DIAG=0" "LSRN_SKETCH_DIAG=1" "LSRN_SKETCH_DIAG=2" "LSRN_SKETCH_DIAG=4" "LSRN_SKETCH_MAXCL=1 LSRN_SKETCH_DIAG=2" "LSRN_SKETCH_MAXCL=1 LSRN_SKETCH_DIAG=4"; do
  env $cfg timeout 300 python tools/diag/sketch_tune.py 100000 2000 2>&1 | tail -1
done | tee gpurun_out/sketch_tune6.jsonl
