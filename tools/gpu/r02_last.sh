#!/bin/bash
# last check of the final tree: pytest -m gpu, smoke(), default bench (3 / 3), t4 bench
mkdir -p gpurun_out/last
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider ) > gpurun_out/last/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/last/pytest_gpu.log; grep -E "passed|failed|rc=" gpurun_out/last/pytest_gpu.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/last/bench.json 2> gpurun_out/last/bench.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/last/bench.json
timeout 900 python bench.py --config t4 --solver cs > gpurun_out/last/bench_t4.json 2> gpurun_out/last/bench_t4.err; echo "t4 rc=$?"; cut -c1-200 gpurun_out/last/bench_t4.json
