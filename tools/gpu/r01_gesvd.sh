#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gesvd or tuning" > gpurun_out/gesvd.log 2>&1; echo "tests rc=$?" >> gpurun_out/gesvd.log
timeout 900 python bench.py --config c4 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e >> gpurun_out/gesvd.log 2>&1
