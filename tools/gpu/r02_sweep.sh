#!/bin/bash
mkdir -p gpurun_out/r02n
timeout 900 python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02n/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02n/pytest.log; tail -3 gpurun_out/r02n/pytest.log
timeout 600 python tools/diag/csr_sketch_modes.py t4 2 > gpurun_out/r02n/t4.jsonl 2>&1; cat gpurun_out/r02n/t4.jsonl
timeout 900 python tools/diag/csr_sketch_modes.py c4 2 > gpurun_out/r02n/c4.jsonl 2>&1; cat gpurun_out/r02n/c4.jsonl
