#!/bin/bash
# run the short bench under several values of an env var: envsweep.sh VAR v1 v2 ...
VAR=$1; shift
for v in "$@"; do
  env $VAR=$v SCG_DEBUG=1 timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/sweep_$v.json 2> gpurun_out/sweep_$v.err
  grep "L2:" gpurun_out/sweep_$v.err
  python3 -c "
import json
d=json.load(open('gpurun_out/sweep_$v.json'))
k=d['kernels']
print('$VAR=$v', round(d['value'],2), ' '.join(f\"{n[:9]}={v['avg_us']:.0f}\" for n,v in k.items()))
"
done
