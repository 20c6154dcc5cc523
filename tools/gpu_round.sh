#!/bin/bash
# One GPU session: tests, bench, ncu launch list, ncu full capture of the top kernel.
# usage: tools/gpu_round.sh <tag> [kernel-regex] [bench args...]
TAG=${1:-r}; KRE=${2:-k_warp_hash}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
fi
timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o $OUT/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > $OUT/ncu_full.log 2>&1
fi
tail -3 $OUT/gpu_tests.log 2>/dev/null; cat $OUT/bench.json; tail -3 $OUT/bench.err
