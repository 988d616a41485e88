#!/bin/bash
# Round 1 measurement pass: smoke, GPU parity, bench (c2), ncu launch list + full captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log | cut -c1-3000
timeout 600 python bench.py --solver cs --no-cpu-baseline > gpurun_out/bench_cs.log 2>&1; echo "bench cs rc=$?"; tail -1 gpurun_out/bench_cs.log | cut -c1-600
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_dense -c 1 -o gpurun_out/prof_sketch $CMD > gpurun_out/ncu_sketch.log 2>&1; echo "ncu sketch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rowpass -s 6 -c 2 -o gpurun_out/prof_rowpass $CMD > gpurun_out/ncu_rowpass.log 2>&1; echo "ncu rowpass rc=$?"
ls -la gpurun_out
