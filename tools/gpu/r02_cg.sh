#!/bin/bash
mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sketch_tall_small or tuning_variants" > gpurun_out/r02/pytest_cg.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_cg.log; tail -3 gpurun_out/r02/pytest_cg.log
timeout 200 python tools/diag/sketch_kernels.py 100000 2000 0 2 > gpurun_out/r02/cg_c2.jsonl 2>&1
timeout 200 python tools/diag/sketch_kernels.py 125000 10000 0 2 > gpurun_out/r02/cg_c5s.jsonl 2>&1
cat gpurun_out/r02/cg_c2.jsonl gpurun_out/r02/cg_c5s.jsonl
