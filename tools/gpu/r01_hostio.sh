#!/bin/bash
# host-IO streaming check: GPU parity tests touching host IO + CSR, then the default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/hostio_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/hostio_tests.log
timeout 600 python bench.py > gpurun_out/hostio_bench_lsqr.json 2> gpurun_out/hostio_bench_lsqr.err
timeout 600 python bench.py --solver cs > gpurun_out/hostio_bench_cs.json 2> gpurun_out/hostio_bench_cs.err
for mb in 64 256; do
  LSRN_HOSTIO_CHUNK_MB=$mb timeout 600 python bench.py --steps 3 > gpurun_out/hostio_bench_mb$mb.json 2>&1
done
tail -3 gpurun_out/hostio_tests.log
