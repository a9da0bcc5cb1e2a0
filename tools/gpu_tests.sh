#!/bin/bash
# GPU call: build, smoke, pytest -m gpu (optionally a -k filter), optional short bench.
TAG=${1:-t}; K=${2:-}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
else
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
fi
if [ -n "$BENCH" ]; then timeout 600 python bench.py $BENCH > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err; fi
