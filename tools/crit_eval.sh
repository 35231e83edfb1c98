# Critical-SM evaluation: parity, then the bench lines it affects; not product code.
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_qr_iterate.py -q -x -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_crit.log 2>&1; tail -1 gpurun_out/pytest_crit.log
ms() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4) if d.get('roofline') else '')"; }
echo "cfg2: $(python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg1: $(python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg1 w96: $(python bench.py --config 1 --window 96 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "hess10k: $(python bench.py --workload hess --n 10000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg3: $(python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
echo "cfg4: $(python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | ms)"
