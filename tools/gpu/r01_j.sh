#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfg in "LSRN_X=0" "LSRN_ROWPASS_KEEP=0" "LSRN_ROWPASS_OCC=2" "LSRN_ROWPASS_OCC=2 LSRN_ROWPASS_KEEP=1"; do
  env $cfg timeout 300 python tools/diag/rowpass_tune.py c2 2>&1 | tail -1
done | tee gpurun_out/rowpass_tune.jsonl
for cfg in "LSRN_X=0" "LSRN_ROWPASS_OCC=2"; do
  env $cfg timeout 300 python tools/diag/rowpass_tune.py c3 2>&1 | tail -1
done | tee -a gpurun_out/rowpass_tune.jsonl
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
