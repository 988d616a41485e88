#!/bin/bash
# bench lines of the other configs (3 timed steps after 3 warm-up) for DESIGN §8
mkdir -p gpurun_out/r02b2
for cfg in "c2 lsqr" "c2 cs" "c3 lsqr" "c4 cs" "t4 cs" "t4 lsqr"; do
  set -- $cfg
  timeout 1200 python bench.py --config $1 --solver $2 --steps 3 --warmup 3 > gpurun_out/r02b2/bench_$1_$2.json 2> gpurun_out/r02b2/bench_$1_$2.err
  echo "$1 $2 rc=$?"; cut -c1-420 gpurun_out/r02b2/bench_$1_$2.json
done
