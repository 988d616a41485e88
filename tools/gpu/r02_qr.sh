#!/bin/bash
# QR route (N = R^-1 when certified full rank): full GPU suite, then the c5 / c4 / c2 bench lines
mkdir -p gpurun_out/r02q
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=10 ) > gpurun_out/r02q/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02q/pytest_gpu.log; tail -16 gpurun_out/r02q/pytest_gpu.log
for cfg in "c5 lsqr" "c4 cs" "c2 lsqr" "c3 lsqr" "t4 cs"; do
  set -- $cfg
  timeout 1500 python bench.py --config $1 --solver $2 --steps 3 --warmup 3 > gpurun_out/r02q/bench_$1_$2.json 2> gpurun_out/r02q/bench_$1_$2.err
  echo "$1 $2 rc=$?"; cut -c1-500 gpurun_out/r02q/bench_$1_$2.json
done
