#!/bin/bash
# GPU call: build, smoke, full pytest -m gpu, default bench (with e2e + cpu baseline)
TAG=${1:-f}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
