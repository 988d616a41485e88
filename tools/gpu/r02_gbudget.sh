mkdir -p gpurun_out
timeout 600 python tools/diag/csr_sketch_gbudget.py t4 -1 1024 256 128 64 32 > gpurun_out/gbudget_t4.jsonl 2>&1
cat gpurun_out/gbudget_t4.jsonl
timeout 600 python tools/diag/csr_sketch_gbudget.py c4 -1 2048 512 128 > gpurun_out/gbudget_c4.jsonl 2>&1
cat gpurun_out/gbudget_c4.jsonl
