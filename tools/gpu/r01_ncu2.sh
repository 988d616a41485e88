#!/bin/bash
mkdir -p gpurun_out/ncu2
O=gpurun_out/ncu2
C1="python tools/diag/rowpass_shape.py 125000 10000 2"
timeout 300 $C1 > $O/c5_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowpass_bulk -s 2 -c 1 -f -o $O/c5_wide1 $C1 > $O/ncu_c5.log 2>&1; echo "c5 rc=$?"
C2="python tools/diag/csr_longpass.py 2000000 4000 cs"
timeout 300 $C2 > $O/csr_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"csr_rowdot_hl8|csr_colgather" -s 4 -c 2 -f -o $O/csr_hl8 $C2 > $O/ncu_csr.log 2>&1; echo "csr rc=$?"
