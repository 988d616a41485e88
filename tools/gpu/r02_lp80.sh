#!/bin/bash
mkdir -p gpurun_out/r02l
for R in 125000 1000000; do
  for il in 0 1; do
    LSRN_OPT_ROWPASS_IL=$il timeout 300 python tools/diag/rowpass_shape.py $R 10000 5 2>&1 | tail -1
  done
done > gpurun_out/r02l/lp_il.jsonl
for il in 0 1; do LSRN_OPT_ROWPASS_IL=$il timeout 300 python tools/diag/rowpass_shape.py 100000 2000 5 2>&1 | tail -1; done >> gpurun_out/r02l/lp_il.jsonl
cat gpurun_out/r02l/lp_il.jsonl
