#!/bin/bash
set -u
mkdir -p gpurun_out/prof
CMD="python bench.py --points 296 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof/plain_b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 2 -c 1 -o gpurun_out/prof/build $CMD > gpurun_out/prof/ncu_build.log 2>&1
echo "build rc=$?"
