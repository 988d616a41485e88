#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py -x -q > gpurun_out/hl8.log 2>&1; echo "tests rc=$?" >> gpurun_out/hl8.log
timeout 300 python tools/diag/csr_longpass.py 2000000 4000 >> gpurun_out/hl8.log 2>&1
LSRN_CSR_ROWDOT_HL2=1 timeout 300 python tools/diag/csr_longpass.py 2000000 4000 >> gpurun_out/hl8.log 2>&1
timeout 300 python tools/diag/csr_longpass.py 2000000 4000 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"csr_rowdot|csr_colgather" -c 6 --csv \
  --log-file gpurun_out/hl8_launches.csv python tools/diag/csr_longpass.py 2000000 4000 > /dev/null 2>&1
