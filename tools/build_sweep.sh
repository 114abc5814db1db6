#!/bin/bash
# A/B of the build kernel's launch configuration: variants built here (python -m
# paper_2305_04318_b200.build --variant NAME -D...), timed on the GPU box with the stage
# timer (C4 and C2 full K).  usage (GPU box): bash tools/build_sweep.sh NAME...
set -u
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v"
  LIK_LIBRARY=paper_2305_04318_b200/liblik_$v.so python tools/bench_configs.py C2 C4 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], 'build_ms', d['stages_ms']['matern_build'], 'chol_ms', d['stages_ms']['chol_fused'], 'pts/s', round(d['points_per_s']))"
done
