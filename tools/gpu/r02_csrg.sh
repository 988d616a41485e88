#!/bin/bash
# stored-G CSR sketch: CSR tests, c4 / t4 sketch times per mode, full-size c4 tests; standalone long pass
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02k/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02k/pytest.log; tail -3 gpurun_out/r02k/pytest.log
timeout 900 python tools/diag/csr_sketch_modes.py c4 2 0 > gpurun_out/r02k/c4.jsonl 2>&1; cat gpurun_out/r02k/c4.jsonl
timeout 600 python tools/diag/csr_sketch_modes.py t4 2 1 > gpurun_out/r02k/t4.jsonl 2>&1; cat gpurun_out/r02k/t4.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c4 or t4" > gpurun_out/r02k/pytest_full.log 2>&1
echo "pytest full rc=$?" >> gpurun_out/r02k/pytest_full.log; tail -3 gpurun_out/r02k/pytest_full.log
LSRN_OPT_ROWPASS_PF=1 timeout 300 python tools/diag/rowpass_shape.py 125000 10000 5 2>&1 | tail -1
