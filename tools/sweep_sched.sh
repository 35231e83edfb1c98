for combo in ${COMBOS:-"24,48,48,0,8|300,0,2" "24,48,32,0,8|300,0,2" "24,32,48,0,8|300,0,2" "24,48,40,0,8|300,0,2" "24,16,48,0,8|300,0,2"}; do
  ch=${combo%|*}; tl=${combo#*|}
  for c in 3 2; do
    echo -n "$ch $tl c$c "
    HQR_CHUNK=$ch HQR_PHASE_TAIL=$tl timeout -s KILL 200 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
  done
done
