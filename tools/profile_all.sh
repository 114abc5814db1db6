#!/bin/bash
# Round profiling pass (under gpurun): plain bench run, launch list of the same
# command, and one `ncu --set full` capture of chol_fused and of build_kernel.
set -u
mkdir -p gpurun_out/prof
# launch list: the bench's own default command (the driver's N = 1 run)
LCMD="python bench.py"
$LCMD > gpurun_out/prof/plain.json 2> gpurun_out/prof/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv $LCMD > /dev/null 2>&1
echo "launches rc=$?"
# full captures: one 592-point launch (2 CTA rounds; replaying a 4,144-point launch
# would save/restore its 68 GB workspace 40 times)
CMD="python bench.py --points 592 --steps 1 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:chol_fused -s 2 -c 1 -o gpurun_out/prof/chol $CMD > gpurun_out/prof/ncu_chol.log 2>&1
echo "chol rc=$?"
ncu --set full --clock-control none --import-source on -k regex:build_kernel -s 2 -c 1 -o gpurun_out/prof/build $CMD > gpurun_out/prof/ncu_build.log 2>&1
echo "build rc=$?"
