#!/bin/bash
# run bench for each variant library; print per-kernel avg_us
for f in paper_1912_02949_b200/lib/variants/*.so; do
  SCG_LIB=$f timeout 300 python bench.py --steps 8 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/var_$(basename $f .so).json 2>/dev/null
  python3 -c "
import json,sys
d=json.load(open('gpurun_out/var_$(basename $f .so).json'))
k=d['kernels']
print('$(basename $f)', round(d['value'],2), ' '.join(f\"{n[:9]}={v['avg_us']:.0f}\" for n,v in k.items()))
"
done
