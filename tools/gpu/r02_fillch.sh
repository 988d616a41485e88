# CSC build with 1024-row chunks for k <= 2048: CSR suite, full-size t4 / c4, sketch times, launch list of the build
# (the 1024-row chunks were an uncommitted experiment, not kept)
mkdir -p gpurun_out/fc
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_multirank_host.py -x -q -p no:cacheprovider > gpurun_out/fc/tests.log 2>&1
tail -1 gpurun_out/fc/tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "t4 or c4" > gpurun_out/fc/full.log 2>&1
tail -1 gpurun_out/fc/full.log
timeout 600 python tools/diag/csr_light_variants.py t4 -1 > gpurun_out/fc/t4.jsonl 2>&1; cat gpurun_out/fc/t4.jsonl
timeout 600 python tools/diag/csr_light_variants.py c4 -1 > gpurun_out/fc/c4.jsonl 2>&1; cat gpurun_out/fc/c4.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"csr_chunk|csr_fill|csr_colptr|excl_scan" --csv \
  --log-file gpurun_out/fc/build_t4.csv python tools/diag/csr_light_variants.py t4 -1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/fc/build_t4.csv > gpurun_out/fc/build_t4.txt 2>&1; grep -E '"kernel"|avg_us' gpurun_out/fc/build_t4.txt | paste - - | head
