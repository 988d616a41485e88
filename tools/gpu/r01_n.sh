#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
./tools/microbench/syevdx_limit 2>&1 | tee gpurun_out/syevdx_limit.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "wide_rows" > gpurun_out/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -5 gpurun_out/pytest_wide.log
for cfg in "LSRN_ROWPASS_ASYNCX=1" "LSRN_ROWPASS_ASYNCX=1 LSRN_ROWPASS_OCC=1"; do
  env $cfg timeout 600 python tools/diag/rowpass_tune.py c5s 2>&1 | tail -1
done | tee gpurun_out/rowpass_tune_c5.jsonl
LSRN_FULLSIZE=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4" > gpurun_out/pytest_full_c4.log 2>&1; echo "pytest c4 rc=$?"; tail -3 gpurun_out/pytest_full_c4.log
