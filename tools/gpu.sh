#!/bin/bash
# run a command on the B200 box from the repo root: tools/gpu.sh <timeout_s> '<command>'
cd /root/repo || exit 1
T=${1:-600}; shift
timeout $((T + 900)) /usr/local/graft/bin/gpurun --timeout "$T" -- "$@" > /tmp/gpurun_last.log 2>&1
rc=$?
tail -2 /tmp/gpurun_last.log
exit $rc
