#!/bin/bash
# quick GPU iteration: selected parity tests, c2 bench (both strategies), optional ncu capture
# usage: tools/iter.sh <tag> [pytest -k expr] [ncu kernel regex]
TAG=$1; K=${2:-"tier or stencil or galerkin"}; KRE=$3
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > $OUT/t.log 2>&1; tail -3 $OUT/t.log
for s in precise hybrid; do
  timeout 200 python bench.py --no-e2e --no-cpu --strategy $s ${BENCH_ARGS} > $OUT/b_$s.json 2>$OUT/b_$s.err
  python -c "
import json; d=json.load(open('$OUT/b_$s.json')); print('$s', d['ms_per_step'], d['value'], {k: [round(x,3) for x in v] for k,v in d['stage_ms'].items()}, d['roofline']['kernel'], d['roofline']['launch_ms'])" || tail -3 $OUT/b_$s.err
done
if [ -n "$KRE" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 2 -c 2 -o $OUT/prof python tools/prof_one.py ${PROF_CFG:-c2} precise > $OUT/ncu.log 2>&1; tail -1 $OUT/ncu.log
fi
