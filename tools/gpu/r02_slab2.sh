#!/bin/bash
mkdir -p gpurun_out/r02
python tools/diag/csr_sketch_variants.py t4 3 > gpurun_out/r02/slab_t4.jsonl 2>&1
python tools/diag/csr_sketch_variants.py c4 1 > gpurun_out/r02/slab_c4.jsonl 2>&1
cat gpurun_out/r02/slab_t4.jsonl gpurun_out/r02/slab_c4.jsonl
