#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python bench.py --config c4 --solver cs --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-3000
