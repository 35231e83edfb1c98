#!/bin/bash
L=$PWD/paper_2007_03576_b200/libhqr_tuning.so
run() { # label env...
  lab=$1; shift
  for c in 2 3; do
    env "$@" HQR_LIB=$L python bench.py --config $c --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tune_$lab_$c.log 2>&1
    python3 -c "import json;d=json.loads(open('gpurun_out/tune_$lab_$c.log').read().strip().splitlines()[-1]);print('$lab cfg$c', round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
}
run base X=1
run chase0 HQR_CHASE_POS=0
run left12 HQR_CHUNK=12,48,48,0,8
run left12n24 HQR_CHUNK=12,24,48,0,8
run bulk96 HQR_CHUNK=24,48,96,0,8
