# c4 long pass: row-pass occupancy (csr_hl_minb) x CSC gather depth
# (the csr_colgather / csr_hl_minb options were an uncommitted experiment, removed after this measurement)
mkdir -p gpurun_out/cg
timeout 600 python -m pytest tests/test_gpu_csr.py -x -q -p no:cacheprovider -k "wide_k or c4" > gpurun_out/cg/tests2.log 2>&1
tail -1 gpurun_out/cg/tests2.log
timeout 900 python tools/diag/longpass_opts.py c4 - csr_hl_minb=3 csr_hl_minb=4 csr_hl_minb=3,csr_colgather=2 > gpurun_out/cg/c4_hl.jsonl 2>&1
cat gpurun_out/cg/c4_hl.jsonl
