#!/bin/bash
# left / near-right phase tails in small chunks: HQR_PHASE_TAIL=ltail,ntail,chunk
CFG=${CFG:-3}
for c in ${TAILS:-"0,0,4" "300,0,4" "600,0,4" "300,150,4" "600,300,2" "1200,300,4" "300,150,8"}; do
  echo -n "$c "
  HQR_PHASE_TAIL=$c python bench.py --config $CFG --no-e2e --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'])"
done
