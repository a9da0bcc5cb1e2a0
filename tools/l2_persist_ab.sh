#!/bin/bash
# SCG_L2_PERSIST: parity (c4 golden), c4 bench A/B, ncu of k_lanczos_a with the window.
TAG=${1:-lp}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
from cuda.bindings import runtime as rt
for a in ('cudaDevAttrMaxPersistingL2CacheSize','cudaDevAttrMaxAccessPolicyWindowSize','cudaDevAttrL2CacheSize'):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
" > $O/attrs.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "config4_real" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for D in 0 1; do
  timeout 600 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu --no-e2e --opts l2_persist=$D > $O/c4_p$D.json 2> $O/c4_p$D.err
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --opts l2_persist=1 > $O/c3_p1.json 2> $O/c3_p1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_a -s 20 -c 1 -o $O/prof_c4p python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e --opts l2_persist=1 > $O/ncu.log 2>&1
echo "ncu exit $?" >> $O/build.log
