#!/bin/bash
# Build in-tree, then run a command on the B200 box via gpurun.  Aborts if the build fails.
# usage: tools/gpu.sh <timeout_s> '<command>'
set -e
cd /root/repo
python -m paper_2305_04318_b200.build > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; echo BUILD FAILED; exit 1; }
python -c "import oracle; oracle.build()"
T=${1:-600}
exec timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "$2"
