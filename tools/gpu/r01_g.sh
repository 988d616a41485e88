#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_g.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/plain_g.log | cut -c1-900
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_g2.log 2>&1 && \
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sketch_ws -c 1 -o gpurun_out/prof_sketch_ws_cl2 $CMD2 > gpurun_out/ncu_ws.log 2>&1; echo "ncu ws rc=$?"
