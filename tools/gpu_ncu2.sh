#!/bin/bash
# build + plain bench + ncu full captures of several kernels (one ncu use)
TAG=${1:-n}; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
$CMD > $O/plain.json 2> $O/plain.err || { echo "plain failed" >> $O/plain.err; exit 1; }
for KRE in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s ${SKIP:-40} -c 1 -o $O/prof_$KRE $CMD > $O/ncu_$KRE.log 2>&1
done
