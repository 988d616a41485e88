#!/bin/bash
mkdir -p gpurun_out/r02
for v in "" "LSRN_OPT_SKETCH_X_L2=1" "LSRN_OPT_SKETCH_NSPLIT=4" "LSRN_OPT_SKETCH_X_L2=1 LSRN_OPT_SKETCH_NSPLIT=4"; do
  env $v timeout 300 python tools/diag/sketch_env.py 1000000 10000 1 2>&1 | tail -1
  env $v timeout 600 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:sketch_ws -c 1 --csv \
     python tools/diag/sketch_env.py 1000000 10000 1 2>&1 | grep dram__bytes | awk -F'","' '{print "  dram_read", $NF}'
done > gpurun_out/r02/l2.txt
cat gpurun_out/r02/l2.txt
