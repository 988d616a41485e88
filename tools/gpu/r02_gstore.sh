#!/bin/bash
# stored-G dense sketch: parity tests, then stage times stored vs in-register on c2 and a c5 shard, then the c5 bench
mkdir -p gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "sketch" > gpurun_out/r02g/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02g/pytest.log; tail -3 gpurun_out/r02g/pytest.log
for v in "" "LSRN_OPT_SKETCH_G=0" "LSRN_OPT_SKETCH_G=2048" "LSRN_OPT_SKETCH_G=16384"; do
  env $v timeout 300 python tools/diag/sketch_env.py 100000 2000 3 2>&1 | tail -1
  env $v timeout 300 python tools/diag/sketch_env.py 125000 10000 2 2>&1 | tail -1
done > gpurun_out/r02g/times.jsonl
cat gpurun_out/r02g/times.jsonl
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r02g/bench_c5.json 2> gpurun_out/r02g/bench_c5.err; echo "bench rc=$?"
cut -c1-900 gpurun_out/r02g/bench_c5.json
