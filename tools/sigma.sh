#!/bin/bash
for sg in 32 64 128 256; do
  SCG_SIGMA=$sg timeout 300 python bench.py --steps 8 --warmup 2 --no-cpu --no-e2e > gpurun_out/sig_$sg.json 2>/dev/null
  python3 -c "
import json
d=json.load(open('gpurun_out/sig_$sg.json'))
k=d['kernels']
print('sigma $sg', round(d['value'],2), ' '.join(f\"{n[:9]}={v['avg_us']:.0f}\" for n,v in k.items()))
"
done
