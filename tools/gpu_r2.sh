#!/bin/bash
# Round-2 GPU call: build, smoke, GPU tests, bench (driver flags), ncu launch list and full captures.
# usage: tools/gpu_r2.sh <tag> [what...]   what: smoke tests bench launches ncu:<regex> full
TAG=${1:-r02}; shift
[ $# -eq 0 ] && set -- smoke tests bench launches
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build exit $?" >> $O/build.log
for w in "$@"; do
  case $w in
    smoke) python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log ;;
    tests) timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log ;;
    tests:*) timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 -k "${w#tests:}" > $O/pytest_gpu_k.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_k.log ;;
    bench) timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err ;;
    ab:*)  # ab:<opts> -- bench with execution options (no cpu / e2e legs)
      OPTS=${w#ab:}; N=${OPTS//[^a-zA-Z0-9_]/_}
      timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --no-e2e --opts "$OPTS" > $O/ab_$N.json 2> $O/ab_$N.err; echo "exit $?" >> $O/ab_$N.err ;;
    abl:*)  # abl:<variant library file under paper_1912_02949_b200/lib/> -- bench with that build
      LIBF=${w#abl:}; N=${LIBF//[^a-zA-Z0-9_]/_}
      SCG_LIB=paper_1912_02949_b200/lib/$LIBF timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --no-e2e > $O/abl_$N.json 2> $O/abl_$N.err; echo "exit $?" >> $O/abl_$N.err ;;
    ncul:*)  # ncul:<variant library>:<kernel regex>:<skip>
      SPEC=${w#ncul:}; LIBF=${SPEC%%:*}; REST=${SPEC#*:}; KRE=${REST%%:*}; SKIP=${REST##*:}
      N=${LIBF//[^a-zA-Z0-9_]/_}_${KRE//[^a-zA-Z0-9_]/_}
      SCG_LIB=paper_1912_02949_b200/lib/$LIBF ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 2 -o $O/prof_$N python bench.py --steps 2 --warmup 5 --no-cpu --no-e2e --no-profile > $O/ncu_full_$N.log 2>&1
      echo "ncu exit $?" >> $O/ncu_full_$N.log ;;
    cfg:*)  # cfg:<config>:<steps>:<opts> -- bench another workload
      SPEC=${w#cfg:}; CFG=${SPEC%%:*}; REST=${SPEC#*:}; STEPS=${REST%%:*}; OPTS=${REST#*:}; [ "$OPTS" = "$REST" ] && OPTS=""
      N=${CFG}_${STEPS}_${OPTS//[^a-zA-Z0-9_]/_}
      timeout 900 python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu --no-e2e --opts "$OPTS" > $O/cfg_$N.json 2> $O/cfg_$N.err; echo "exit $?" >> $O/cfg_$N.err ;;
    ncuc:*)  # ncuc:<config>:<kernel regex>:<skip>
      SPEC=${w#ncuc:}; CFG=${SPEC%%:*}; REST=${SPEC#*:}; KRE=${REST%%:*}; SKIP=${REST##*:}
      N=${CFG}_${KRE//[^a-zA-Z0-9_]/_}
      ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 -o $O/prof_$N python bench.py --config $CFG --steps 2 --warmup 60 --no-cpu --no-e2e --no-profile > $O/ncu_full_$N.log 2>&1
      echo "ncu exit $?" >> $O/ncu_full_$N.log ;;
    cfgnp:*)  # cfgnp:<config>:<steps>:<opts> -- as cfg, without per-kernel events (launch-bound graphs)
      SPEC=${w#cfgnp:}; CFG=${SPEC%%:*}; REST=${SPEC#*:}; STEPS=${REST%%:*}; OPTS=${REST#*:}; [ "$OPTS" = "$REST" ] && OPTS=""
      N=${CFG}_${STEPS}_${OPTS//[^a-zA-Z0-9_]/_}
      timeout 900 python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu --no-e2e --no-profile --opts "$OPTS" > $O/cfgnp_$N.json 2> $O/cfgnp_$N.err; echo "exit $?" >> $O/cfgnp_$N.err ;;
    benchnocpu) timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err ;;
    full) timeout 900 python bench.py --steps 997 --warmup 3 --no-cpu --no-e2e > $O/bench_full.json 2> $O/bench_full.err; echo "exit $?" >> $O/bench_full.err ;;
    ref) timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref exit $?" >> $O/ref.err ;;
    launches)
      CMD="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e"
      $CMD > $O/plain.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
      echo "ncu launches exit $?" >> $O/plain.log ;;
    ncu:*)  # ncu:<kernel regex>:<launches to skip>
      SPEC=${w#ncu:}; KRE=${SPEC%%:*}; SKIP=${SPEC##*:}; [ "$SKIP" = "$SPEC" ] && SKIP=60
      N=${KRE//[^a-zA-Z0-9_]/_}
      CMD="python bench.py --steps 2 --warmup 5 --no-cpu --no-e2e --no-profile"
      ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 -o $O/prof_$N $CMD > $O/ncu_full_$N.log 2>&1
      echo "ncu full exit $?" >> $O/ncu_full_$N.log
      # text pages for reading here (the merge back is capped at 64 MiB: keep the report compressed)
      ncu -i $O/prof_$N.ncu-rep --page raw --csv > $O/prof_${N}_raw.csv 2>/dev/null
      ncu -i $O/prof_$N.ncu-rep --page details --csv > $O/prof_${N}_details.csv 2>/dev/null
      ncu -i $O/prof_$N.ncu-rep --page source --csv > $O/prof_${N}_source.csv 2>/dev/null
      gzip -f $O/prof_$N.ncu-rep ;;
  esac
done
echo done > $O/DONE
