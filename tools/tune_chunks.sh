#!/bin/bash
# fused-kernel task chunk sizes: left,near,bulk,tail,tail_chunk
for c in ${CHUNKS:-"12,6,24,1200,6" "12,6,32,1600,6" "12,6,24,2000,8" "16,6,32,2000,8" "12,4,24,1200,4" "10,6,20,1500,5"}; do
  echo -n "$c "
  HQR_CHUNK=$c python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'])"
done
