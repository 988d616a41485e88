#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_csr.py -q > gpurun_out/pytest_csr.log 2>&1; echo "pytest csr rc=$?"; tail -4 gpurun_out/pytest_csr.log
timeout 600 python bench.py --config t4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_t4.log 2>&1; echo "bench t4 rc=$?"; tail -1 gpurun_out/bench_t4.log | cut -c1-700
