#!/bin/bash
# SCG_ELL_DEEP: parity tests + c4 bench A/B + c3 bench (unchanged path) + ncu of the deep c4 SpMV.
TAG=${1:-ed}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "ell_deep or config4 or ell_ or small_and_ragged or config3_bench" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/c3.json 2> $O/c3.err
for D in 0 1; do
  timeout 600 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu --no-e2e --opts ell_deep=$D > $O/c4_d$D.json 2> $O/c4_d$D.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_a -s 20 -c 1 -o $O/prof_c4deep python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --opts ell_deep=1 > $O/ncu.log 2>&1
echo "ncu exit $?" >> $O/build.log
