#!/bin/bash
# what the driver runs at round end: pytest -m gpu (with -x), the bench at 20 steps / 5 warm-up,
# and the reference arm
mkdir -p gpurun_out/r02d
( time timeout 1500 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=15 ) > gpurun_out/r02d/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d/pytest_gpu.log; tail -22 gpurun_out/r02d/pytest_gpu.log
( time timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
echo "bench rc=$?"; tail -4 gpurun_out/r02d/bench.err
( time timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02d/ref.json 2> gpurun_out/r02d/ref.err
echo "ref rc=$?"; tail -4 gpurun_out/r02d/ref.err
