#!/bin/bash
# same-box K1 timing of whole trees under abtrees/<rev> (each with its own binding + library) and this tree
REPS=${1:-1}; SEEDS=${2:-256}
ROOT=$(pwd)
for r in $(seq 1 $REPS); do
  for d in abtrees/* .; do
    (cd "$d" && timeout 300 python bench.py --seeds $SEEDS --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
      > /tmp/abt.json 2>/dev/null; python -c "import json; d=json.load(open('/tmp/abt.json')); print('$d', $r, round(d['phase_ms']['k1_simulate'],1))" >> "$ROOT/gpurun_out/abt_summary.txt" 2>&1)
  done
done
