#!/bin/bash
# ncu --set full of k_lanczos_a on configs[4] and configs[2] (bench launch configuration).
TAG=${1:-c42}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in c4 c2; do
  CMD="python bench.py --config $C --steps 3 --warmup 3 --no-cpu --no-e2e"
  timeout 600 $CMD > $O/bench_$C.json 2> $O/bench_$C.err
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_a -s 20 -c 1 -o $O/prof_$C $CMD > $O/ncu_$C.log 2>&1
  echo "$C ncu exit $?" >> $O/build.log
done
