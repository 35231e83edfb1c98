# window-side sweep at configs[3] and configs[2] (the product default is 96)
mkdir -p gpurun_out
ms() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config']['window'])"; }
for w in 96 64 80 88 104 112 96; do
  echo "cfg3 w$w $(timeout 300 python bench.py --window $w --steps 4 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
  echo "cfg2 w$w $(timeout 300 python bench.py --config 2 --window $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
done
