#!/bin/bash
mkdir -p gpurun_out/r02
python tools/diag/c18_floor.py 250 1000 2000 4100 9000 > gpurun_out/r02/c18_floor.jsonl 2> gpurun_out/r02/c18_floor.err
( time python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r02/ref_c5.json 2> gpurun_out/r02/ref_c5.err
cat gpurun_out/r02/c18_floor.jsonl; cat gpurun_out/r02/ref_c5.json; tail -4 gpurun_out/r02/ref_c5.err
