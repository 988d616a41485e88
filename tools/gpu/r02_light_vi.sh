# light kernel with two sketch rows per thread: parity tests + t4 / c4 sketch times
# (the 10xx csr_light values were an uncommitted experiment, removed after this measurement)
mkdir -p gpurun_out/vi
timeout 900 python -m pytest tests/test_gpu_csr.py -x -q -p no:cacheprovider -k "light_kernel or sketch_vs_oracle or full" > gpurun_out/vi/tests.log 2>&1
tail -1 gpurun_out/vi/tests.log
timeout 600 python tools/diag/csr_light_variants.py t4 -1 1018 1014 1028 1048 > gpurun_out/vi/t4.jsonl 2>&1; cat gpurun_out/vi/t4.jsonl
timeout 600 python tools/diag/csr_light_variants.py c4 -1 1048 1088 1044 > gpurun_out/vi/c4.jsonl 2>&1; cat gpurun_out/vi/c4.jsonl
