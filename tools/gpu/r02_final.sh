#!/bin/bash
# CSR slab unroll check (t4, c4) + the default bench's launch list and DRAM traffic (post-chunking)
mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_csr.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02f/pytest_csr.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f/pytest_csr.log; tail -2 gpurun_out/r02f/pytest_csr.log
timeout 600 python tools/diag/csr_sketch_variants.py t4 5 > gpurun_out/r02f/slab_t4.jsonl 2>&1; cat gpurun_out/r02f/slab_t4.jsonl
timeout 900 python tools/diag/csr_sketch_variants.py c4 2 > gpurun_out/r02f/slab_c4.jsonl 2>&1; cat gpurun_out/r02f/slab_c4.jsonl
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sketch|rowpass|colreduce|lsqr|csr_|fill_kernel|copy_scale|transpose|extract_r|form_nt|check_finite|build_jw" --csv \
  --log-file gpurun_out/r02f/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02f/ncu_launch.log 2>&1
echo "ncu rc=$?"
