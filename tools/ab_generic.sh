#!/bin/bash
# same-box K1 timing: LEAN specialisation vs --generic (inside gpurun): tools/ab_generic.sh [seeds] [reps]
SEEDS=${1:-256}; REPS=${2:-2}
for r in $(seq 1 $REPS); do for V in lean generic; do
  X=""; [ $V = generic ] && X="--generic"
  timeout 300 python bench.py --seeds $SEEDS --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $X > gpurun_out/abg_${V}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/abg_${V}_$r.json')); print('$V', $r, round(d['phase_ms']['k1_simulate'],1))" >> gpurun_out/abg_summary.txt
done; done
