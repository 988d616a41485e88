#!/bin/bash
mkdir -p gpurun_out/r02
for v in "" "LSRN_OPT_SKETCH_MAXCL=2" "LSRN_OPT_SKETCH_TILE=0" "LSRN_OPT_SKETCH_TILE=0 LSRN_OPT_SKETCH_MAXCL=1"; do
  env $v timeout 300 python tools/diag/sketch_env.py 125000 10000 2 2>&1 | tail -1
  env $v timeout 300 python tools/diag/sketch_env.py 100000 2000 3 2>&1 | tail -1
done > gpurun_out/r02/cl.txt
cat gpurun_out/r02/cl.txt
