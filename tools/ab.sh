#!/bin/bash
# A/B bench of library variants on the GPU box (run under gpurun):
#   tools/ab.sh POINTS lib1 lib2 ...   (lib = path to a built liblik variant)
P=$1; shift
for rep in 1 2; do
  for L in "$@"; do
    LIK_LIBRARY=$L python bench.py --points $P --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/ab.json'))
print('$L', round(d['value'],1), 'chol TF', round(d['roofline']['achieved'],2), 'frac', round(d['roofline']['frac'],4), 'build ms', round(d['stages_ms_per_step']['matern_build'],2), 'clk', d['clocks']['sm_mhz'])"
  done
done
