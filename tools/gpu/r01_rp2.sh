#!/bin/bash
mkdir -p gpurun_out
for shape in "20000 20000" "125000 10000"; do
for ws in 2048 2560 3334 4096 5000; do
  for occ in 1 2; do
    LSRN_ROWPASS_WIDE_SLICE=$ws LSRN_ROWPASS_OCC=$occ timeout 120 python tools/diag/rowpass_shape.py $shape >> gpurun_out/rp2.log 2>&1 || echo "FAILED $shape $ws $occ" >> gpurun_out/rp2.log
  done
done
done
