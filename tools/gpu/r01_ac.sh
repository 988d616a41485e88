#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_csr.py -q -x > gpurun_out/pytest_csr.log 2>&1; echo "pytest csr rc=$?"; tail -3 gpurun_out/pytest_csr.log
timeout 300 python tools/diag/csr_sketch_time.py 2>&1 | tail -3
