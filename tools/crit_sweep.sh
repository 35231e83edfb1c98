# Critical-SM / near-task order sweep (tuning build); not product code.
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_crit.log 2>&1; tail -1 gpurun_out/pytest_crit.log
L=$PWD/paper_2007_03576_b200/libhqr_tuning.so
ms() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"; }
for o in 0 1; do for c in 0 22; do
  echo "cfg2 near_order $o crit $c: $(HQR_NEAR_ORDER=$o HQR_CRIT_SMS=$c HQR_LIB=$L python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
done; done
echo "cfg2 default: $(python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg3 default: $(python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg3 order0: $(HQR_NEAR_ORDER=0 HQR_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
