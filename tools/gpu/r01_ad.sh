#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py --smoke > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -15 gpurun_out/memcheck.log
