#!/bin/bash
# One GPU call: tests, bench, ncu launch list + full capture of the top kernel.
# usage: tools/gpu_round.sh <tag> [kernel-regex]
TAG=${1:-r01}; KRE=${2:-k_lanczos_a}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu1 exit $?" >> $O/plain.log
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 40 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu2 exit $?" >> $O/plain.log
