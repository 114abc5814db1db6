#!/bin/bash
# one `ncu --set full` capture of chol_fused on a 2-wave bench run (under gpurun)
set -u
mkdir -p gpurun_out/prof
CMD="python bench.py --points 592 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof/plain.json 2> gpurun_out/prof/plain.err && \
ncu --set full --clock-control none --import-source on -k regex:chol_fused -s 2 -c 1 -o gpurun_out/prof/chol $CMD > gpurun_out/prof/ncu_chol.log 2>&1
echo "chol rc=$?"
