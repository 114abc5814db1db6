#!/bin/bash
# Phase-0 box facts: FP64 peaks + clocks under FP64 load.
set -u
OUT=gpurun_out/phase0
mkdir -p $OUT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $OUT/clocks.csv &
SMI=$!
./tools/phase0/fp64_peaks > $OUT/fp64_peaks.jsonl 2>&1
kill $SMI
nproc > $OUT/host.txt; lscpu | grep "Model name" >> $OUT/host.txt
cat $OUT/fp64_peaks.jsonl
