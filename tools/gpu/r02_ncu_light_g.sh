# ncu --set full of one stored-G CSR light-sketch launch on t4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_sketch_light_g -s 1 -c 1 \
  -o gpurun_out/ncu_light_g_t4 -f python tools/diag/csr_sketch_modes.py t4 2 > gpurun_out/ncu_light_g.log 2>&1
tail -3 gpurun_out/ncu_light_g.log
