#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_rows" > gpurun_out/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -5 gpurun_out/pytest_wide.log
for cfg in "LSRN_ROWPASS_ASYNCX=1" "LSRN_ROWPASS_ASYNCX=0"; do
  env $cfg timeout 600 python tools/diag/rowpass_tune.py c5s 2>&1 | tail -1
done | tee gpurun_out/rowpass_tune_c5.jsonl
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
LSRN_FULLSIZE=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c4" > gpurun_out/pytest_full_c3c4.log 2>&1; echo "pytest c3c4 rc=$?"; tail -5 gpurun_out/pytest_full_c3c4.log
