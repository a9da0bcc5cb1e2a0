#!/bin/bash
# In-flow pass-1 figure: the bench-configuration test, a short and the default bench.
O=gpurun_out/${1:-fl}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bench_launch_configuration or config3_first or steps_resume" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_short.json 2> $O/bench_short.err; echo "exit $?" >> $O/bench_short.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
