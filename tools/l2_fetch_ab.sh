#!/bin/bash
# L2 fetch granularity A/B on c4 and c3 (bench, no cpu / e2e legs) + ncu DRAM bytes of c4 k_lanczos_a at 32 B.
TAG=${1:-lf}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for G in 0 32 64 128; do
  timeout 600 python tools/l2_fetch_ab.py $G --config c4 --steps 6 --warmup 3 --no-cpu --no-e2e > $O/c4_g$G.json 2> $O/c4_g$G.err
done
for G in 0 32; do
  timeout 300 python tools/l2_fetch_ab.py $G --steps 20 --warmup 5 --no-cpu --no-e2e > $O/c3_g$G.json 2> $O/c3_g$G.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k_lanczos_a -s 20 -c 1 --csv python tools/l2_fetch_ab.py 32 --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_c4_g32.csv 2> $O/ncu.err
echo "ncu exit $?" >> $O/build.log
