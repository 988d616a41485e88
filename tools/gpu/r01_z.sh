#!/bin/bash
# measurement pass: smoke, gpu tests, bench c2 (all legs), CS, reference, launch list, ncu full top kernels; c5 bench + full test
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_z.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_z.log | cut -c1-300
timeout 300 python bench.py --solver cs --no-cpu-baseline > gpurun_out/bench_z_cs.log 2>&1; echo "bench cs rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_z_ref.log 2>&1; echo "ref rc=$?"
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > gpurun_out/plain_z2.log 2>&1 && \
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_z.csv $CMD2 > gpurun_out/ncu_list_z.log 2>&1; echo "ncu list rc=$?"
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sketch_ws -c 1 -o gpurun_out/prof_z_sketch $CMD2 > gpurun_out/ncu_z1.log 2>&1; echo "ncu sk rc=$?"
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rowpass_bulk -s 4 -c 2 -o gpurun_out/prof_z_rowpass $CMD2 > gpurun_out/ncu_z2.log 2>&1; echo "ncu rp rc=$?"
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_z_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_z_c5.log | cut -c1-600
timeout 900 python bench.py --config c5 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_z_c5_cs.log 2>&1; echo "bench c5 cs rc=$?"
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_z_c3.log 2>&1; echo "bench c3 rc=$?"
LSRN_FULLSIZE=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5" > gpurun_out/pytest_full_c5.log 2>&1; echo "pytest c5 rc=$?"; tail -3 gpurun_out/pytest_full_c5.log
