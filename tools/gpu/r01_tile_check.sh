#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tile_check.log 2>&1; echo "tests rc=$?" >> gpurun_out/tile_check.log
timeout 600 python bench.py > gpurun_out/tile_bench_lsqr.json 2> gpurun_out/tile_bench_lsqr.err
tail -3 gpurun_out/tile_check.log
