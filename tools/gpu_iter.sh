#!/bin/bash
# GPU iteration call: build, quick parity subset, bench (c3), optional ncu of one kernel.
# usage: gpu_iter.sh TAG [KERNEL_REGEX]
TAG=${1:-it}; KRE=${2:-}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYK:-config0_full or sharded_config1 or small_and_ragged or config3 or apply_D or heavy}" > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
CMD="python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
$CMD > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
if [ -n "$KRE" ]; then
  CMD2="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
  $CMD2 > $O/plain.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$KRE -s ${SKIP:-40} -c 1 -o $O/prof $CMD2 > $O/ncu_full.log 2>&1
  echo "ncu exit $?" >> $O/bench.err
fi
