#!/bin/bash
mkdir -p gpurun_out/r02
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sketch_tall_small or solve_c1" > gpurun_out/r02/pytest_bmint.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_bmint.log; tail -4 gpurun_out/r02/pytest_bmint.log
timeout 200 python tools/diag/sketch_kernels.py 100000 2000 0 > gpurun_out/r02/bmint_c2.jsonl 2>&1
timeout 300 python tools/diag/sketch_kernels.py 125000 10000 0 > gpurun_out/r02/bmint_c5s.jsonl 2>&1
cat gpurun_out/r02/bmint_c2.jsonl gpurun_out/r02/bmint_c5s.jsonl
