#!/bin/bash
# A/B of environment settings in one GPU session: tools/abenv.sh <tag> <cfg> "<env1>" "<env2>" ...
TAG=$1; CFG=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for e in "$@"; do
  env $e timeout 300 python bench.py --config $CFG --strategy ${ST:-precise} --no-e2e --no-cpu --no-per-config --steps 5 > $OUT/ab.json 2> $OUT/ab.err
  python -c "
import json; d=json.load(open('$OUT/ab.json')); print('$CFG', '$e', d['ms_per_step'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()}, {k:{c:v for c,v in x.items() if v>0.5} for k,x in d.get('class_ms',{}).items()})" || tail -2 $OUT/ab.err
done; done
