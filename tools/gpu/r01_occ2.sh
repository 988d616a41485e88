#!/bin/bash
mkdir -p gpurun_out
LSRN_ROWPASS_OCC=2 LSRN_ROWPASS_BUDGET_KB=110 timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/occ2.jsonl 2>&1 || echo FAILED >> gpurun_out/occ2.jsonl
LSRN_ROWPASS_OCC=2 LSRN_ROWPASS_BUDGET_KB=110 LSRN_ROWPASS_WIDE_SLICE=5120 timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/occ2.jsonl 2>&1 || echo FAILED >> gpurun_out/occ2.jsonl
timeout 300 python tools/diag/rowpass_tune.py c5s >> gpurun_out/occ2.jsonl 2>&1
