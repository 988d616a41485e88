mkdir -p gpurun_out
./tools/microbench/svd_bench 4000 2000 1800 > gpurun_out/svd_2000.jsonl 2>&1; cat gpurun_out/svd_2000.jsonl
./tools/microbench/svd_bench 400 200 200 2>&1 | tail -4
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log | cut -c1-1500
