#!/bin/bash
# PDL trigger placement A/B on c3 and c0 (no profiling events: they break the programmatic chains)
for v in early late; do
  for p in 1 0; do
    for cfg in c3 c0; do
      SCG_PDL=$p SCG_LIB=paper_1912_02949_b200/lib/variants/$v.so timeout 600 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/pl_${v}_${p}_$cfg.json 2>/dev/null
      python3 -c "
import json; d=json.loads(open('gpurun_out/pl_${v}_${p}_$cfg.json').readline()); print('$v pdl=$p $cfg', round(d['value'],2))" >> gpurun_out/pdl_late.txt
    done
  done
done
