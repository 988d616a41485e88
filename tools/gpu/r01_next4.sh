#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/next4/gamma_sweep.py > gpurun_out/next4_gamma_sweep.jsonl 2> gpurun_out/next4_gamma_sweep.err
FIG1_RUNS=5 timeout 1500 python tools/next4/fig1_cond_iters.py > gpurun_out/next4_fig1.jsonl 2> gpurun_out/next4_fig1.err
tail -2 gpurun_out/next4_gamma_sweep.err gpurun_out/next4_fig1.err
