#!/bin/bash
# stored-G sketch: launch list with DRAM bytes of one c5 bench step, and a full ncu capture of one
# sketch_ws_kernel launch (and the generator) on a c5-shaped shard
mkdir -p gpurun_out/r02h
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"sketch|rowpass|colreduce|lsqr|fill_kernel|copy_scale|transpose|extract_r|form_nt|check_finite|build_jw" --csv \
  --log-file gpurun_out/r02h/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02h/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sketch_ws_kernel|sketch_gen_g" -c 2 \
  -o gpurun_out/r02h/sketch_g python tools/diag/sketch_env.py 125000 10000 1 > gpurun_out/r02h/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/r02h/ncu_full.log
