#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config t4 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_t4.log 2>&1; echo "bench t4 rc=$?"; tail -1 gpurun_out/bench_t4.log | cut -c1-1500
timeout 600 python bench.py --config t4 --solver cs --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_t4_cs.log 2>&1; echo "bench t4 cs rc=$?"; tail -1 gpurun_out/bench_t4_cs.log | cut -c1-600
