#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "wide_rows or tuning" > gpurun_out/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -3 gpurun_out/pytest_wide.log
for cfg in "LSRN_ROWPASS_ASYNCX=1" "LSRN_ROWPASS_ASYNCX=0"; do
  env $cfg timeout 600 python tools/diag/rowpass_tune.py c5s 2>&1 | tail -1
done | tee gpurun_out/rowpass_tune_c5.jsonl
timeout 300 python tools/microbench/dgemm_probe.py && \
timeout 300 ncu --profile-from-start off --set full --clock-control none -c 1 -o gpurun_out/prof_dgemm python tools/microbench/dgemm_probe.py > gpurun_out/ncu_dgemm.log 2>&1; echo "ncu dgemm rc=$?"
