#!/bin/bash
# full measurement pass: smoke, tests, bench (c2 LSQR default line, CS), launch list, ncu full of top kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_k.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_k.log | cut -c1-400
timeout 600 python bench.py --solver cs --no-cpu-baseline > gpurun_out/bench_k_cs.log 2>&1; echo "bench cs rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_k_ref.log 2>&1; echo "bench ref rc=$?"; tail -1 gpurun_out/bench_k_ref.log | cut -c1-300
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_k2.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k.csv $CMD2 > gpurun_out/ncu_list_k.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sketch_ws -c 1 -o gpurun_out/prof_k_sketch $CMD2 > gpurun_out/ncu_k1.log 2>&1; echo "ncu sk rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rowpass_bulk -s 4 -c 2 -o gpurun_out/prof_k_rowpass $CMD2 > gpurun_out/ncu_k2.log 2>&1; echo "ncu rp rc=$?"
