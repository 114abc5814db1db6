#!/bin/bash
# One GPU-box pass: full -m gpu suite, smoke, the default bench line, the C5 bench line,
# the bench under a one-rank NCCL group, and the ncu launch list of the default bench.
# usage (GPU box): bash tools/round_check.sh TAG
set -u
T=${1:-r02}
mkdir -p gpurun_out/$T
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/$T/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$T/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$T/smoke.log
python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_c5.json 2> gpurun_out/$T/bench_c5.err
python bench.py --dist --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_dist.json 2> gpurun_out/$T/bench_dist.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/ncu_bench.log 2>&1
python tools/ktimes_summary.py gpurun_out/$T/launches.csv > gpurun_out/$T/launch_shares.txt
tail -3 gpurun_out/$T/gputest.log; tail -2 gpurun_out/$T/smoke.log; cat gpurun_out/$T/launch_shares.txt
