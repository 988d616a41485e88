#!/bin/bash
mkdir -p gpurun_out/r02
for pf in 0 1 2 3 4; do
  LSRN_OPT_ROWPASS_PF=$pf timeout 200 python tools/diag/rowpass_shape.py 125000 10000 5 2>&1 | tail -1
done > gpurun_out/r02/pf_c5.jsonl
for pf in 0 2; do
  LSRN_OPT_ROWPASS_PF=$pf timeout 200 python tools/diag/rowpass_shape.py 20000 20000 5 2>&1 | tail -1
  LSRN_OPT_ROWPASS_PF=$pf timeout 200 python tools/diag/rowpass_shape.py 100000 2000 5 2>&1 | tail -1
done >> gpurun_out/r02/pf_c5.jsonl
cat gpurun_out/r02/pf_c5.jsonl
timeout 300 python -m pytest tests/test_gpu_rowpass.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "rowpass or wide_rows or solve_c1" 2>&1 | tail -2
