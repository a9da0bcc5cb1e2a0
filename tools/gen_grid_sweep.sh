#!/bin/bash
# Side-stream start-vector draw: grid size sweep on c3 (bench, no cpu / e2e legs).
TAG=${1:-gg}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for G in ${GRIDS:-0 8 16 32 74 148}; do
  SCG_GEN_GRID=$G timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/g$G.json 2> $O/g$G.err
done
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:k_monitor -s 2 -c 1 -o $O/prof_mon $CMD2 > $O/ncu_mon.log 2>&1
echo "ncu exit $?" >> $O/build.log
