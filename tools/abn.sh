#!/bin/bash
# same-box timing of several prebuilt libraries: tools/abn.sh "A B C" [seeds] [reps]  (inside gpurun)
LIBS=${1:-"A B"}; SEEDS=${2:-256}; REPS=${3:-2}
for r in $(seq 1 $REPS); do for L in $LIBS; do
  SDAS_LIB=$PWD/paper_2601_03197_b200/libsdas_$L.so timeout 300 python bench.py --seeds $SEEDS --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/ab_${L}_$r.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/ab_${L}_$r.json')); print('$L', $r, round(d['phase_ms']['k1_simulate'],1))" >> gpurun_out/ab_summary.txt
done; done
