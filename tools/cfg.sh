#!/bin/bash
# quick timing of configs (bench lines, no e2e/cpu).  usage: tools/cfg.sh <tag> <cfg...>
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${TESTK:-tier or galerkin or stencil}" > $OUT/t.log 2>&1; tail -1 $OUT/t.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 5 > $OUT/$c.json 2> $OUT/$c.err
  python -c "
import json; d=json.load(open('$OUT/$c.json')); print('$c', d['ms_per_step'], d['value'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()})" || tail -2 $OUT/$c.err
done
