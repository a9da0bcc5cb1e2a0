for v in late; do for p in 1 0; do for cfg in c1 c2; do
  SCG_PDL=$p SCG_LIB=paper_1912_02949_b200/lib/variants/$v.so timeout 600 python bench.py --config $cfg --steps 300 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/pl_${v}_${p}_$cfg.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/pl_${v}_${p}_$cfg.json').readline()); print('$v pdl=$p $cfg', round(d['value'],2))" >> gpurun_out/pdl_late2.txt
done; done; done
SCG_PDL=1 SCG_LIB=paper_1912_02949_b200/lib/variants/late.so timeout 900 python bench.py --no-cpu --no-e2e --no-profile > gpurun_out/pl_late_full.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/pl_late_full.json').readline()); print('late pdl=1 c3 full', round(d['value'],2))" >> gpurun_out/pdl_late2.txt
