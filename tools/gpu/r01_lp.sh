#!/bin/bash
mkdir -p gpurun_out
for kb in 192 224; do
  LSRN_ROWPASS_BUDGET_KB=$kb timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/lp.jsonl 2>&1
done
timeout 300 python tools/diag/csr_longpass.py 2000000 4000 >> gpurun_out/lp.jsonl 2>&1
timeout 300 python tools/diag/csr_longpass.py 2000000 4000 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csr_|rowpass|colreduce|lsqr|krylov" -c 60 --csv \
  --log-file gpurun_out/lp_csr_launches.csv python tools/diag/csr_longpass.py 2000000 4000 > /dev/null 2>&1
echo done >> gpurun_out/lp.jsonl
