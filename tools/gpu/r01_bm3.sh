#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/diag/sketch_tune.py 100000 2000 > gpurun_out/bm3.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_csr.py -x -q >> gpurun_out/bm3.jsonl 2>&1
timeout 300 python tools/diag/csr_sketch_time.py >> gpurun_out/bm3.jsonl 2>&1
