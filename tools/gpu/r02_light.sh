# stored-G CSR light kernel defaults: CSR tests, full-size t4 / c4 tests, sketch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr.py -x -q -p no:cacheprovider > gpurun_out/light_tests.log 2>&1
tail -2 gpurun_out/light_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "t4 or c4" > gpurun_out/light_full.log 2>&1
tail -2 gpurun_out/light_full.log
timeout 600 python tools/diag/csr_light_variants.py t4 -1 > gpurun_out/light3_t4.jsonl 2>&1; cat gpurun_out/light3_t4.jsonl
timeout 600 python tools/diag/csr_light_variants.py c4 -1 > gpurun_out/light3_c4.jsonl 2>&1; cat gpurun_out/light3_c4.jsonl
