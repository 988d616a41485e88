# ncu --set full of the pipelined CSR single pass (variant 10) on t4
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_rowdot_all_pipe -s 3 -c 1 \
  -o gpurun_out/ncu_csr_all_v10 -f python tools/diag/csr_all_variants.py t4 10 > gpurun_out/ncu_csr_all.log 2>&1
tail -3 gpurun_out/ncu_csr_all.log
