#!/bin/bash
# quick parity subset for every variant library
for f in paper_1912_02949_b200/lib/variants/*.so; do
  SCG_LIB=$f timeout 600 python -m pytest tests -m gpu -x -q -k "config0_full or sharded_config1 or small_and_ragged or heavy or config2_first or breakdown" > gpurun_out/vp_$(basename $f .so).log 2>&1
  echo "$(basename $f) $(tail -n 1 gpurun_out/vp_$(basename $f .so).log)"
done
