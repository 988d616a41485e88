#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu.log
for cfg in "LSRN_SKETCH_MAXCL=1" "LSRN_SKETCH_MAXCL=2" "LSRN_SKETCH_MAXCL=4" "LSRN_SKETCH_V1=1"; do
  env $cfg timeout 300 python tools/diag/sketch_tune.py 100000 2000 2>&1 | tail -1
done | tee gpurun_out/sketch_tune2.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_o.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_o.log | cut -c1-700
LSRN_FULLSIZE=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c4" > gpurun_out/pytest_full_c3c4.log 2>&1; echo "pytest c3c4 rc=$?"; tail -3 gpurun_out/pytest_full_c3c4.log
