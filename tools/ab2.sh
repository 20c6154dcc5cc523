#!/bin/bash
# A/B of in-tree builds in one GPU session: tools/ab2.sh <tag> "<libs>" "<cfgs>" [strategy]
TAG=$1; LIBS=$2; CFGS=$3; ST=${4:-precise}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for c in $CFGS; do for lib in $LIBS; do
  SPGEMM_LIB=$lib timeout 300 python bench.py --config $c --strategy $ST --no-e2e --no-cpu --no-per-config --steps 5 > $OUT/ab_${c}_${lib}_$rep.json 2> $OUT/ab_${c}_${lib}_$rep.err
  python -c "
import json; d=json.load(open('$OUT/ab_${c}_${lib}_$rep.json')); print('$c', '$lib', d['ms_per_step'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()}, d.get('class_ms'))" || tail -2 $OUT/ab_${c}_${lib}_$rep.err
done; done; done
