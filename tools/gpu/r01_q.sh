#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for cfg in "LSRN_SKETCH_MAXCL=2" "LSRN_SKETCH_MAXCL=2 LSRN_SKETCH_DIAG=1" "LSRN_SKETCH_MAXCL=1 LSRN_SKETCH_DIAG=1"; do
  env $cfg timeout 300 python tools/diag/sketch_tune.py 100000 2000 2>&1 | tail -1
done | tee gpurun_out/sketch_tune3.jsonl
CMD2="python tools/diag/sketch_tune.py 100000 2000"
timeout 300 $CMD2 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:sketch_ws -s 3 -c 1 -o gpurun_out/prof_ws_bm2 $CMD2 > gpurun_out/ncu_ws3.log 2>&1; echo "ncu rc=$?"
