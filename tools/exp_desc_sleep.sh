mkdir -p gpurun_out
ms() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
for v in base ds32 ds128; do
  echo "cfg3 $v $(HQR_LIB=$PWD/tools/libhqr_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
  echo "cfg2 $v $(HQR_LIB=$PWD/tools/libhqr_$v.so timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
done; done
