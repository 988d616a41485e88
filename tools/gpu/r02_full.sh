#!/bin/bash
# round 2: full-size parity tests + the default bench (c5) + its launch list
mkdir -p gpurun_out/r02
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider --durations=20 \
  > gpurun_out/r02/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_full.log
python bench.py > gpurun_out/r02/bench_c5.json 2> gpurun_out/r02/bench_c5.err
echo "bench rc=$?" >> gpurun_out/r02/bench_c5.err
tail -30 gpurun_out/r02/pytest_full.log; tail -3 gpurun_out/r02/bench_c5.err; cat gpurun_out/r02/bench_c5.json
