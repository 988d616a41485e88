#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/diag/csr_diag.py 2>&1 | tail -20
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_d.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/plain_d.log | cut -c1-900
