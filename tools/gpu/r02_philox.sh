#!/bin/bash
# experiment: the dense sketch with Philox only (Box-Muller replaced by a bit cast; timing only)
mkdir -p gpurun_out/r02
cp paper_1109_5981_b200/liblsrn.so /tmp/liblsrn_real.so
cp tools/exp/liblsrn_philoxonly.so paper_1109_5981_b200/liblsrn.so
timeout 200 python tools/diag/sketch_kernels.py 125000 10000 0 > gpurun_out/r02/rng_philoxonly.jsonl 2>&1
cp /tmp/liblsrn_real.so paper_1109_5981_b200/liblsrn.so
cat gpurun_out/r02/rng_philoxonly.jsonl
