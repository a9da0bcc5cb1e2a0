#!/bin/bash
# summarize a gpu_iter.sh output directory
O=gpurun_out/$1
tail -n 2 $O/smoke.log; tail -n 3 $O/pytest_gpu.log; grep -v Remark $O/bench.err | tail -n 4
python3 -c "
import json,sys
d=json.load(open('$O/bench.json')); print('it/s', round(d['value'],2), 'frac', round(d['roofline']['frac'],3))
for k,v in d['kernels'].items(): print(f\"  {k:24s} {v['launches']:6d} {v['avg_us']:9.1f} us {v['gbs']:8.1f} GB/s share {v['share']:.3f}\")
" 2>/dev/null
[ -f $O/prof.ncu-rep ] && python3 tools/ncu_summary.py $O/prof.ncu-rep
