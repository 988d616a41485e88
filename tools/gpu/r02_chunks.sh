#!/bin/bash
mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sketch_tall_small or tuning_variants" > gpurun_out/r02/pytest_chunks.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_chunks.log; tail -2 gpurun_out/r02/pytest_chunks.log
for v in "LSRN_OPT_SKETCH_CHUNKS=0" "" "LSRN_OPT_SKETCH_CHUNKS=16 LSRN_OPT_SKETCH_X_L2=1"; do
  env $v timeout 300 python tools/diag/sketch_env.py 1000000 10000 1 2>&1 | tail -1
  env $v timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:sketch_ws --csv \
     python tools/diag/sketch_env.py 1000000 10000 1 2>&1 | grep dram__bytes | awk -F'","' '{s+=$NF} END {print "  dram_read_total", s}'
done > gpurun_out/r02/chunks.txt
cat gpurun_out/r02/chunks.txt
