#!/bin/bash
# Round-2 evidence session: GPU tests, default bench line (per_config block), ncu launch list of
# the same command (c2 only), ncu full capture of c2's dominant kernels.
# usage: tools/r2_session.sh <tag> ; SKIP_TESTS=1 SKIP_NCU=1 KRE=regex
TAG=${1:-s}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TTIME:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 ${PYK:+-k "$PYK"} > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
  tail -40 $OUT/gpu_tests.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 1200 python bench.py $BENCH_ARGS > $OUT/bench.json 2> $OUT/bench.err; echo BENCH_RC=$?
  cat $OUT/bench.json | head -c 6000; tail -5 $OUT/bench.err
fi
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-per-config $BENCH_ARGS > $OUT/ncu_launches.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_bw_sym|k_bwrow}" -s ${KSKIP:-6} -c ${KCOUNT:-2} -o $OUT/full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-per-config $BENCH_ARGS > $OUT/ncu_full.log 2>&1
  echo NCU done; tail -3 $OUT/ncu_full.log
fi
