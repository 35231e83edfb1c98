# confirmation: window 88 vs 96 at n = 10000 (configs[2], hess_n) and n = 4000 (configs[1]), alternating
ms() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['config']['window'])"; }
for rep in 1 2 3; do for w in 96 88; do
  echo "cfg2 w$w $(timeout 200 python bench.py --config 2 --window $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
done; done
for w in 96 88; do
  echo "hess w$w $(timeout 200 python bench.py --workload hess --window $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
  echo "cfg1 w$w $(timeout 200 python bench.py --config 1 --window $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
done
