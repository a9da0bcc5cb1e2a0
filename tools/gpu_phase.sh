#!/bin/bash
# Phase retrieval GPU call: build, quick timing, tests, ncu captures of the FFT kernels.
# usage: tools/gpu_phase.sh <tag> [what...]   what: quick:<n>:<T> tests ncu:<regex>:<n>:<T>:<skip>
TAG=${1:-p}; shift
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build exit $?" >> $O/build.log
for w in "$@"; do
  case $w in
    quick:*) S=${w#quick:}; N=${S%%:*}; R1=${S#*:}; T=${R1%%:*}; FL=${R1#*:}; [ "$FL" = "$R1" ] && FL=0
      timeout 600 python tools/phase_quick.py $N $T $FL > $O/quick_${N}_${T}_${FL}.log 2>&1 ;;
    tests) timeout 1500 python -m pytest tests/test_gpu_phase.py -q -x --durations=20 > $O/pytest_phase.log 2>&1; echo "pytest exit $?" >> $O/pytest_phase.log ;;
    ncu:*) S=${w#ncu:}; KRE=${S%%:*}; R1=${S#*:}; N=${R1%%:*}; R2=${R1#*:}; T=${R2%%:*}; SKIP=${R2#*:}
      NM=${KRE//[^a-zA-Z0-9_]/_}_$N
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 -o $O/prof_$NM python tools/phase_quick.py $N $T > $O/ncu_$NM.log 2>&1
      ncu -i $O/prof_$NM.ncu-rep --page details > $O/prof_${NM}_details.txt 2>/dev/null
      ncu -i $O/prof_$NM.ncu-rep --page raw --csv > $O/prof_${NM}_raw.csv 2>/dev/null
      ncu -i $O/prof_$NM.ncu-rep --page source --csv > $O/prof_${NM}_source.csv 2>/dev/null
      gzip -f $O/prof_$NM.ncu-rep ;;
  esac
done
echo done > $O/DONE
