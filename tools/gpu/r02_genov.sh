mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_csr.py -x -q -p no:cacheprovider -k "overlap or stored or sketch_vs_oracle" > gpurun_out/genov_tests.log 2>&1
tail -2 gpurun_out/genov_tests.log
timeout 900 python tools/diag/csr_gen_overlap.py t4 c4 0 1 2 4 8 > gpurun_out/genov2.jsonl 2>&1
cat gpurun_out/genov2.jsonl
