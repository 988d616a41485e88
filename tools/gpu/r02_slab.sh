#!/bin/bash
mkdir -p gpurun_out/r02
python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02/pytest_csr.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_csr.log
tail -5 gpurun_out/r02/pytest_csr.log
python tools/diag/csr_sketch_variants.py t4 3 > gpurun_out/r02/slab_t4.jsonl 2>&1
python tools/diag/csr_sketch_variants.py c4 2 > gpurun_out/r02/slab_c4.jsonl 2>&1
python tools/diag/svd_methods.py c5 jw polar > gpurun_out/r02/svd_c5.jsonl 2>&1
python tools/diag/svd_methods.py c4 polar > gpurun_out/r02/svd_c4.jsonl 2>&1
cat gpurun_out/r02/slab_t4.jsonl gpurun_out/r02/slab_c4.jsonl gpurun_out/r02/svd_c5.jsonl gpurun_out/r02/svd_c4.jsonl
