#!/bin/bash
# Full ncu capture of ONE K1 launch (tools/profile_k1.py) + summary; run inside gpurun from the repo root.
# usage: tools/ncu_k1.sh <config> <seeds> <tag>   -> gpurun_out/<tag>.ncu-rep, <tag>_summary.json, <tag>.log
CFG=${1:-2}; SEEDS=${2:-64}; TAG=${3:-k1}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k1_simulate -c 1 \
  -o gpurun_out/$TAG -f python tools/profile_k1.py --config $CFG --seeds $SEEDS > gpurun_out/$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep gpurun_out/$TAG.log gpurun_out/${TAG}_summary.json config-$CFG \
  >> gpurun_out/$TAG.log 2>&1
