#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_c.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/plain_c.log | cut -c1-2500
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c.csv $CMD2 > gpurun_out/ncu_list_c.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rowpass_bulk -s 2 -c 2 -o gpurun_out/prof_rowpass_bulk $CMD2 > gpurun_out/ncu_rp.log 2>&1; echo "ncu rp rc=$?"
