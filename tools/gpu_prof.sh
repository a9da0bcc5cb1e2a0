#!/bin/bash
# GPU call: build, short bench (c3), then ncu --set full of one kernel.  usage: gpu_prof.sh TAG REGEX [SKIP]
TAG=${1:-p}; KRE=${2:-k_lanczos_a}; SKIP=${3:-40}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
$CMD > $O/plain.json 2> $O/plain.err && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "exit $?" >> $O/plain.err
