#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "lambda_path or wide_rows" > gpurun_out/pytest_path.log 2>&1; echo "pytest path rc=$?"; tail -3 gpurun_out/pytest_path.log
for cfg in "LSRN_X=0" "LSRN_ROWPASS_OCC=2 LSRN_ROWPASS_WIDE_SLICE=4096" "LSRN_ROWPASS_OCC=2 LSRN_ROWPASS_WIDE_SLICE=2560" "LSRN_ROWPASS_OCC=1 LSRN_ROWPASS_WIDE_SLICE=4096" "LSRN_ROWPASS_OCC=1 LSRN_ROWPASS_WIDE_SLICE=10000"; do
  env $cfg timeout 120 python tools/diag/rowpass_tune.py c5s 2>&1 | tail -1
done | tee gpurun_out/rowpass_tune_c5b.jsonl
