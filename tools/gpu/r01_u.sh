#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sketch" > gpurun_out/pytest_sk.log 2>&1; echo "pytest sketch rc=$?"; tail -3 gpurun_out/pytest_sk.log
for cfg in "LSRN_SKETCH_MAXCL=2" "LSRN_SKETCH_MAXCL=1" "LSRN_SKETCH_MAXCL=4" "LSRN_SKETCH_DIAG=1"; do
  env $cfg timeout 300 python tools/diag/sketch_tune.py 100000 2000 2>&1 | tail -1
done | tee gpurun_out/sketch_tune7.jsonl
timeout 300 python tools/diag/sketch_tune.py 200000 4096 2>&1 | tail -1 | tee -a gpurun_out/sketch_tune7.jsonl
