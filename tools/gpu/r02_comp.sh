#!/bin/bash
# compensated mode (precision = 1) + regressions of the passes it shares the loop with; t4/c4 slab on the C15 recipe
mkdir -p gpurun_out/r02c
timeout 1200 python -m pytest tests/test_gpu_compensated.py tests/test_gpu_parity.py tests/test_gpu_csr.py tests/test_gpu_abi_contract.py -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/r02c/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c/pytest.log; tail -14 gpurun_out/r02c/pytest.log
timeout 600 python tools/diag/compensated_cost.py > gpurun_out/r02c/comp_cost.jsonl 2>&1; cat gpurun_out/r02c/comp_cost.jsonl
timeout 600 python tools/diag/csr_sketch_variants.py t4 5 > gpurun_out/r02c/slab_t4.jsonl 2>&1; cat gpurun_out/r02c/slab_t4.jsonl
