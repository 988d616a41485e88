#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
./tools/microbench/svd_bench2 4000 2000 1800 > gpurun_out/svd2_c2.jsonl 2>&1; echo "svd2 rc=$?"; cat gpurun_out/svd2_c2.jsonl
./tools/microbench/svd_bench2 400 200 200 > gpurun_out/svd2_small.jsonl 2>&1; tail -12 gpurun_out/svd2_small.jsonl
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_b.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "lsrn_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv $CMD > gpurun_out/ncu_list_b.log 2>&1; echo "ncu list rc=$?"
tail -1 gpurun_out/plain_b.log | cut -c1-2500
