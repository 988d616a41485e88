#!/bin/bash
mkdir -p gpurun_out/r02k
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"csr_" --csv \
  --log-file gpurun_out/r02k/launches_c4.csv python tools/diag/csr_sketch_modes.py c4 2 > gpurun_out/r02k/ncu_c4.log 2>&1
echo "ncu rc=$?"
timeout 900 python tools/diag/iter_vs_gmode.py > gpurun_out/r02k/iter_gmode.jsonl 2>&1; cat gpurun_out/r02k/iter_gmode.jsonl
