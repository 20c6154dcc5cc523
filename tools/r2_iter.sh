#!/bin/bash
# round-2 iteration: GPU tests (parity first, then full-size configs), bench lines per config.
# usage: tools/r2_iter.sh <tag> [pytest -k expr] ; BENCH_CFGS="c2 c3b" STRATS="precise hybrid"
TAG=$1; K=${2:-""}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
free -g > $OUT/free.txt; nproc >> $OUT/free.txt
if [ -n "$K" ]; then
  timeout ${TTIME:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" --durations=15 > $OUT/t.log 2>&1
  tail -25 $OUT/t.log
fi
for c in ${BENCH_CFGS:-}; do
  for s in ${STRATS:-precise}; do
    timeout 600 python bench.py --config $c --strategy $s --no-e2e --no-cpu --no-per-config --steps 5 > $OUT/b_${c}_$s.json 2> $OUT/b_${c}_$s.err
    python -c "
import json; d=json.load(open('$OUT/b_${c}_$s.json')); print('$c $s', d['ms_per_step'], d['value'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()}, d['roofline']['kernel'], d['roofline']['launch_ms'])" || tail -3 $OUT/b_${c}_$s.err
  done
done
