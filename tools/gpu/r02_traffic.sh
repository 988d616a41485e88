# DRAM bytes per kernel of one bench step (warm-up + 1 timed solve) for c2, t4, c4 -> traffic.json entries
# (the first run had no -k filter and profiled every torch kernel of the t4 / c4 data generators: only c2 finished)
mkdir -p gpurun_out/tr
for cfg in c2 t4 c4; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"sketch|rowpass|csr_|colreduce|gen_g" \
    --log-file gpurun_out/tr/launches_$cfg.csv python bench.py --config $cfg --solver cs --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/tr/ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
  python tools/ncu_summary.py dram gpurun_out/tr/launches_$cfg.csv > gpurun_out/tr/dram_$cfg.json 2>&1; head -c 1500 gpurun_out/tr/dram_$cfg.json; echo
done
