#!/bin/bash
# experiment: the dense sketch with the RNG replaced by constants (timing only; wrong results)
mkdir -p gpurun_out/r02
timeout 200 python tools/diag/sketch_kernels.py 125000 10000 0 > gpurun_out/r02/rng_on.jsonl 2>&1
cp paper_1109_5981_b200/liblsrn.so /tmp/liblsrn_real.so
cp tools/exp/liblsrn_norng.so paper_1109_5981_b200/liblsrn.so
timeout 200 python tools/diag/sketch_kernels.py 125000 10000 0 > gpurun_out/r02/rng_off.jsonl 2>&1
cp /tmp/liblsrn_real.so paper_1109_5981_b200/liblsrn.so
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:sketch_ws -c 1 --csv \
   python tools/diag/sketch_kernels.py 125000 10000 0 > gpurun_out/r02/ncu_raster.csv 2>&1
cat gpurun_out/r02/rng_on.jsonl gpurun_out/r02/rng_off.jsonl; grep -E "dram__|duration|pipe" gpurun_out/r02/ncu_raster.csv | awk -F'","' '{print $(NF-2), $NF}'
