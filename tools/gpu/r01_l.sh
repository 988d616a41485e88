#!/bin/bash
# large configs: c3, c5 (80 GB), c4 (CSR) full-size parity + one bench line each; cuBLAS DGEMM probe
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
free -g | head -2; nproc
LSRN_FULLSIZE=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c5" > gpurun_out/pytest_full_c3c5.log 2>&1; echo "pytest c3c5 rc=$?"; tail -5 gpurun_out/pytest_full_c3c5.log
timeout 1200 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-1500
timeout 1200 python bench.py --config c5 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_cs.log 2>&1; echo "bench c5 cs rc=$?"
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
LSRN_FULLSIZE=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4" > gpurun_out/pytest_full_c4.log 2>&1; echo "pytest c4 rc=$?"; tail -5 gpurun_out/pytest_full_c4.log
timeout 2400 python bench.py --config c4 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"; tail -1 gpurun_out/bench_c4.log | cut -c1-1500
