#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rowpass.py tests/test_gpu_parity.py -q -x > gpurun_out/cr.log 2>&1; echo "tests rc=$?" >> gpurun_out/cr.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e >> gpurun_out/cr.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > /dev/null 2>&1 && timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cr_launches.csv $CMD2 > /dev/null 2>&1
