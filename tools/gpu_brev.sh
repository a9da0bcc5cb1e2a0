#!/bin/bash
# k_lanczos_b reversed chunked traversal: parity subset, A/B (short window), default bench.
O=gpurun_out/${1:-br}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q -k "config1_trajectory or ell_ or config3 or bench_launch or steps_resume or small_and_ragged or config4" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for v in 0 1 0 1; do
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --no-e2e --opts b_ascending=$v > $O/ab_asc$v.$RANDOM.json 2>> $O/ab.err
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
