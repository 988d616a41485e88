#!/bin/bash
mkdir -p gpurun_out/r02
python tools/diag/t4_sketch_once.py t4 > gpurun_out/r02/t4_once.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:csr_sketch_slab -c 1 \
    -o gpurun_out/r02/ncu_slab_t4 -f python tools/diag/t4_sketch_once.py t4 > gpurun_out/r02/ncu_slab_t4.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r02/ncu_slab_t4.log
