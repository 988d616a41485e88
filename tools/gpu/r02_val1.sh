#!/bin/bash
# after the pipelined CSR single pass: full GPU suite + t4 bench lines
mkdir -p gpurun_out/r02v
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=10 ) > gpurun_out/r02v/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02v/pytest_gpu.log; tail -16 gpurun_out/r02v/pytest_gpu.log
for s in lsqr cs; do
  timeout 900 python bench.py --config t4 --solver $s --steps 3 --warmup 3 > gpurun_out/r02v/bench_t4_$s.json 2> gpurun_out/r02v/bench_t4_$s.err
  echo "t4 $s rc=$?"; cat gpurun_out/r02v/bench_t4_$s.json | head -c 600; echo
done
