#!/bin/bash
# round-2 closing run: the driver's steps (pytest -m gpu, bench 20/5 on the default c5, the
# reference arm) and bench lines of c2 / c3 / c4 / t4 (3 timed steps after 3 warm-up)
mkdir -p gpurun_out/r02z
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=10 ) > gpurun_out/r02z/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02z/pytest_gpu.log; tail -4 gpurun_out/r02z/pytest_gpu.log
for cfg in "c4 cs" "t4 cs" "t4 lsqr" "c2 lsqr" "c3 lsqr"; do
  set -- $cfg
  timeout 1200 python bench.py --config $1 --solver $2 --steps 3 --warmup 3 > gpurun_out/r02z/bench_$1_$2.json 2> gpurun_out/r02z/bench_$1_$2.err
  echo "$1 $2 rc=$?"; cut -c1-200 gpurun_out/r02z/bench_$1_$2.json
done
( time timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02z/bench.json 2> gpurun_out/r02z/bench.err
echo "bench rc=$?"; cut -c1-300 gpurun_out/r02z/bench.json; tail -3 gpurun_out/r02z/bench.err
( time timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02z/ref.json 2> gpurun_out/r02z/ref.err
echo "ref rc=$?"; cut -c1-300 gpurun_out/r02z/ref.json; tail -3 gpurun_out/r02z/ref.err
