#!/bin/bash
mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sketch_tall_small or tiles_and_clusters or wide_rows" > gpurun_out/r02/pytest_raster.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_raster.log; tail -2 gpurun_out/r02/pytest_raster.log
timeout 200 python tools/diag/sketch_kernels.py 100000 2000 0 > gpurun_out/r02/raster_c2.jsonl 2>&1
timeout 300 python tools/diag/sketch_kernels.py 1000000 10000 0 > gpurun_out/r02/raster_c5.jsonl 2>&1
cat gpurun_out/r02/raster_c2.jsonl gpurun_out/r02/raster_c5.jsonl
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:sketch_ws -c 1 --csv \
   python tools/diag/sketch_kernels.py 1000000 10000 0 2>&1 | grep -E "dram__bytes|duration" | cut -c1-250
timeout 300 ./tools/microbench/svd_bench5 10000 > gpurun_out/r02/svd5.jsonl 2>&1; cat gpurun_out/r02/svd5.jsonl
