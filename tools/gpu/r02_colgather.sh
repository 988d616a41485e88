# c4 long pass: CSC-gather entries in flight (csr_colgather), parity tests, ncu of the two kernels
# (the csr_colgather / csr_hl_minb options were an uncommitted experiment, removed after this measurement)
mkdir -p gpurun_out/cg
timeout 600 python -m pytest tests/test_gpu_csr.py -x -q -p no:cacheprovider -k "wide_k or c4" > gpurun_out/cg/tests.log 2>&1
tail -1 gpurun_out/cg/tests.log
timeout 900 python tools/diag/longpass_opts.py c4 - csr_colgather=2 csr_colgather=4 csr_colgather=8 > gpurun_out/cg/c4.jsonl 2>&1
cat gpurun_out/cg/c4.jsonl
timeout 900 ncu --set full --clock-control none -k regex:"csr_rowdot_hl8|csr_colgather" -s 40 -c 2 \
  -o gpurun_out/cg/ncu_c4_lp -f python tools/diag/longpass_opts.py c4 - > gpurun_out/cg/ncu.log 2>&1
tail -2 gpurun_out/cg/ncu.log
