#!/bin/bash
# round-1 measurement pass: smoke, gpu tests, bench legs per config, launch list, ncu full of the top kernels
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c2_lsqr.json 2> $O/bench_c2_lsqr.err; echo "bench rc=$?"
timeout 600 python bench.py --solver cs > $O/bench_c2_cs.json 2> $O/bench_c2_cs.err; echo "bench cs rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_c2_reference.json 2> $O/bench_c2_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_lsqr.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config t4 --no-cpu-baseline > $O/bench_t4_lsqr.json 2> $O/bench_t4.err; echo "t4 rc=$?"
timeout 600 python bench.py --config t4 --solver cs --no-cpu-baseline > $O/bench_t4_cs.json 2> $O/bench_t4_cs.err; echo "t4 cs rc=$?"
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > $O/plain.log 2>&1 && \
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_lsqr.csv $CMD2 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:sketch_ws -c 1 -o $O/prof_sketch $CMD2 > $O/ncu_sk.log 2>&1; echo "ncu sk rc=$?"
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:rowpass_bulk -s 4 -c 2 -o $O/prof_rowpass $CMD2 > $O/ncu_rp.log 2>&1; echo "ncu rp rc=$?"
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5_lsqr.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c5 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5_cs.json 2> $O/bench_c5_cs.err; echo "c5 cs rc=$?"
timeout 900 python bench.py --config c4 --solver cs --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c4_cs.json 2> $O/bench_c4_cs.err; echo "c4 cs rc=$?"
