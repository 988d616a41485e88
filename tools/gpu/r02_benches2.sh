#!/bin/bash
# final bench lines of c2 / c3 / c4 / t4 (3 timed steps after 3 warm-up), and an ncu capture of an
# in-solve c5 long pass (graph node) next to the same kernel launched directly
mkdir -p gpurun_out/r02b3
for cfg in "c2 lsqr" "c2 cs" "c3 lsqr" "c4 cs" "t4 cs" "t4 lsqr"; do
  set -- $cfg
  timeout 1200 python bench.py --config $1 --solver $2 --steps 3 --warmup 3 > gpurun_out/r02b3/bench_$1_$2.json 2> gpurun_out/r02b3/bench_$1_$2.err
  echo "$1 $2 rc=$?"; cut -c1-300 gpurun_out/r02b3/bench_$1_$2.json
done
timeout 900 ncu --set full --graph-profiling node --clock-control none -k regex:rowpass_bulk --launch-skip 40 -c 3 \
  -o gpurun_out/r02b3/lp_graph python tools/diag/lp_insolve.py > gpurun_out/r02b3/ncu_lp.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r02b3/ncu_lp.log
