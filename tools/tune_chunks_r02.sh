#!/bin/bash
# fused-kernel task chunk sizes after the K-loop change (tuning build via HQR_LIB): left,near,bulk,tail,tail_chunk
# prints ms per sweep, the SM clock and ms x clock (cycles, comparable across power-capped runs)
for rep in 1 2; do
for c in "24,48,48,0,8" "24,48,96,0,8" "48,48,96,0,8" "24,48,32,0,8" "16,32,48,0,8" "32,64,64,0,8"; do
  echo -n "$c "
  HQR_CHUNK=$c python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); m=d['ms_per_step']; c=d['clocks']['sm_mhz']; print(round(m,2), c, round(m*c/1000,1))"
done
done
