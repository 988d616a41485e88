#!/bin/bash
# sustained DMMA and cuBLAS DGEMM throughput with clocks (the c5 sketch runs 14 s)
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 200 > gpurun_out/r02/smi_sustained.csv &
SMI=$!
./tools/microbench/fp64_sustained 12 > gpurun_out/r02/fp64_sustained.jsonl
python - >> gpurun_out/r02/fp64_sustained.jsonl <<'PY'
import json, time, torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
torch.matmul(a, b); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
n = 0; t = time.time(); e0.record()
while time.time() - t < 12:
    torch.matmul(a, b); n += 1
    if n % 10 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"test": "cublas_dgemm_sustained", "n": 8192, "launches": n, "seconds": ms / 1e3,
                  "tflops": 2 * 8192 ** 3 * n / ms / 1e9}))
PY
kill $SMI
tail -2 gpurun_out/r02/fp64_sustained.jsonl
python - <<'PY'
import statistics
rows = [l.strip().split(", ") for l in open("gpurun_out/r02/smi_sustained.csv") if l.strip()]
clk = [float(r[0]) for r in rows if float(r[1]) > 400]
print("clock median under load", statistics.median(clk) if clk else None, "samples", len(clk),
      "power_cap_active", sum(1 for r in rows if r[2].strip() == "Active"))
PY
