#!/bin/bash
mkdir -p gpurun_out/r02h2
timeout 900 python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02h2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h2/pytest.log; tail -3 gpurun_out/r02h2/pytest.log
timeout 900 python tools/diag/csr_sketch_modes.py c4 2 > gpurun_out/r02h2/c4.jsonl 2>&1
LSRN_OPT_CSR_HEAVY_FMA=1 timeout 900 python tools/diag/csr_sketch_modes.py c4 2 >> gpurun_out/r02h2/c4.jsonl 2>&1
cat gpurun_out/r02h2/c4.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c4" > gpurun_out/r02h2/pytest_full.log 2>&1
echo "pytest full rc=$?" >> gpurun_out/r02h2/pytest_full.log; tail -2 gpurun_out/r02h2/pytest_full.log
