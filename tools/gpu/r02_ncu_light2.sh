# t4 sketch after the light-kernel change: launch list (times, DRAM) + full capture of one light launch
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:csr_ --csv \
  --log-file gpurun_out/t4_sketch_launches.csv python tools/diag/csr_light_variants.py t4 -1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/t4_sketch_launches.csv > gpurun_out/t4_sketch_launches.txt 2>&1; head -30 gpurun_out/t4_sketch_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_sketch_light_g -s 20 -c 1 \
  -o gpurun_out/ncu_light_g2_t4 -f python tools/diag/csr_light_variants.py t4 -1 > gpurun_out/ncu_light_g2.log 2>&1
tail -2 gpurun_out/ncu_light_g2.log
