#!/bin/bash
# round 2: GPU tests except the full-size ones (tests/test_gpu_fullsize.py runs separately)
mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py -p no:cacheprovider \
  --durations=25 > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
tail -40 gpurun_out/r02/pytest_gpu.log
