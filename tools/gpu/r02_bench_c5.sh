#!/bin/bash
# the default bench (c5) + its launch list (our kernels) + DRAM traffic of the sketch and long pass
mkdir -p gpurun_out/r02b
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r02b/bench_c5.json 2> gpurun_out/r02b/bench_c5.err
echo "bench rc=$?"; cat gpurun_out/r02b/bench_c5.json | cut -c1-600
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
  -k regex:"sketch|rowpass|colreduce|lsqr|csr_|fill_kernel|copy_scale|transpose|extract_r|form_nt|check_finite|build_jw" --csv \
  --log-file gpurun_out/r02b/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02b/ncu_launch.log 2>&1
echo "ncu rc=$?"
