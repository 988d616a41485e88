# after pruning the CSR single-pass variants: CSR suite, smoke(), t4 bench line
mkdir -p gpurun_out/post
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_abi_contract.py -x -q -p no:cacheprovider > gpurun_out/post/tests.log 2>&1
tail -1 gpurun_out/post/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/post/smoke.log 2>&1; tail -2 gpurun_out/post/smoke.log
timeout 600 python tools/diag/csr_all_variants.py t4 0 6 10 > gpurun_out/post/csr_all.jsonl 2>&1; cat gpurun_out/post/csr_all.jsonl
