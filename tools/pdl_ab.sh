#!/bin/bash
# A/B of programmatic dependent launch, with and without per-kernel events
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for prof in "--no-profile" ""; do for pdl in 0 1; do
  SCG_PDL=$pdl timeout 600 python bench.py --steps ${STEPS:-300} --warmup 3 --no-cpu --no-e2e $prof ${BENCH_ARGS} > gpurun_out/pdl_$pdl$prof.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('gpurun_out/pdl_$pdl$prof.json')); print('pdl=$pdl prof=\"$prof\"', round(d['value'],3), round(d['ms_per_step'],3))"
done; done
