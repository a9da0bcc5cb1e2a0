#!/bin/bash
for c in ${CFGS:-c2 c3}; do for dyn in 0 1; do
  SCG_DYN=$dyn timeout 600 python bench.py --config $c --steps ${STEPS:-60} --warmup 3 --no-cpu --no-e2e > gpurun_out/dyn_${c}_$dyn.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('gpurun_out/dyn_${c}_$dyn.json')); print('$c dyn=$dyn', round(d['value'],2), round(d['kernels']['lanczos_a_spmv_dot']['avg_us'],1))"
done; done
