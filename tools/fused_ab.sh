#!/bin/bash
# fused pass-1 kernel A/B per config (no profiling events)
rm -f gpurun_out/fused_ab.txt
for cfg in c0 c1 c2 c3; do
  st=300; [ $cfg = c3 ] && st=60
  for f in 0 1; do
    SCG_FUSED=$f timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/fab_${cfg}_$f.json 2>/dev/null
    python3 -c "
import json; d=json.loads(open('gpurun_out/fab_${cfg}_$f.json').readline()); print('$cfg SCG_FUSED=$f', round(d['value'],2), 'it/s')" >> gpurun_out/fused_ab.txt
  done
done
