#!/bin/bash
# fused-kernel task chunk sizes: left,near,bulk,tail,tail_chunk
for c in ${CHUNKS:-"12,6,24,1200,6" "16,8,32,1200,6" "24,8,48,1500,6" "24,12,48,2000,8" "32,12,64,2000,8" "12,6,48,1500,6" "24,6,24,1200,6"}; do
  echo -n "$c "
  HQR_CHUNK=$c python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'])"
done
