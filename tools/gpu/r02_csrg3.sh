#!/bin/bash
mkdir -p gpurun_out/r02k
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"csr_" --csv \
  --log-file gpurun_out/r02k/launches_c4_v2.csv python tools/diag/csr_sketch_modes.py c4 2 > gpurun_out/r02k/ncu_c4_v2.log 2>&1
echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"csr_" --csv \
  --log-file gpurun_out/r02k/launches_t4_v2.csv python tools/diag/csr_sketch_modes.py t4 2 > gpurun_out/r02k/ncu_t4_v2.log 2>&1
echo "ncu rc=$?"
