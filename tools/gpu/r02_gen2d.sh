# generators without per-pair 64-bit division: parity tests + sketch stage times
mkdir -p gpurun_out/gen2d
timeout 900 python -m pytest tests/test_gpu_csr.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/gen2d/tests.log 2>&1
tail -2 gpurun_out/gen2d/tests.log
timeout 600 python tools/diag/csr_light_variants.py t4 -1 > gpurun_out/gen2d/t4.jsonl 2>&1; cat gpurun_out/gen2d/t4.jsonl
timeout 600 python tools/diag/csr_light_variants.py c4 -1 > gpurun_out/gen2d/c4.jsonl 2>&1; cat gpurun_out/gen2d/c4.jsonl
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gen2d/c2.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/gen2d/c2.json').read().splitlines()[-1]); print('c2', d['value'], d['stages_s'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gen_g --csv --log-file gpurun_out/gen2d/gen_launches.csv \
  python tools/diag/csr_light_variants.py t4 -1 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/gen2d/gen_launches.csv 2>&1 | grep -A4 gen_g | head -8
