#!/bin/bash
# round 2 validation: every GPU test (full-size included), the default bench (c5) and the
# other configs' bench lines, the launch list and the DRAM traffic of the c5 step
mkdir -p gpurun_out/r02v
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/r02v/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02v/pytest_gpu.log
tail -45 gpurun_out/r02v/pytest_gpu.log | tail -8
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r02v/bench_c5.json 2> gpurun_out/r02v/bench_c5.err
echo "bench c5 rc=$?"
for c in c2 t4 c4; do
  timeout 900 python bench.py --config $c --solver cs --steps 3 --warmup 3 > gpurun_out/r02v/bench_${c}_cs.json 2> gpurun_out/r02v/bench_${c}_cs.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c2 --solver lsqr --steps 3 --warmup 3 > gpurun_out/r02v/bench_c2_lsqr.json 2> gpurun_out/r02v/bench_c2_lsqr.err
timeout 900 python bench.py --config t4 --solver lsqr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02v/bench_t4_lsqr.json 2> gpurun_out/r02v/bench_t4_lsqr.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02v/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/r02v/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --profile-from-start off -k regex:"sketch_ws|rowpass_bulk" -c 3 --csv --log-file gpurun_out/r02v/traffic_c5.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02v/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
