# CSR single-pass variants on t4 (tools/diag/csr_all_variants.py) and their parity tests
# (variants 4, 5, 7, 8, 9, 11, 12, 13 were removed after this measurement; 0, 6, 10 remain)
mkdir -p gpurun_out
timeout 600 python tools/diag/csr_all_variants.py t4 0 6 10 11 12 13 > gpurun_out/csr_all_t4_ts.jsonl 2>&1
cat gpurun_out/csr_all_t4_ts.jsonl
timeout 900 python -m pytest tests/test_gpu_csr.py -x -q -k "single_pass" > gpurun_out/csr_all_tests.log 2>&1
tail -3 gpurun_out/csr_all_tests.log
