#!/bin/bash
# Session: GPU tests (subset by KSEL, all by default) + c2 / g3d27 hybrid one-walk vs two-walk vs precise.
OUT=gpurun_out/${TAG:-r2f}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${KSEL:+-k "$KSEL"} > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -3 $OUT/tests.log
for rep in 1 2; do for c in ${CFGS:-c2 g3d27}; do
  for v in "hybrid 0" "hybrid 1" "precise 0"; do set -- $v
    SPGEMM_BW_TWO_WALK=$2 timeout 300 python bench.py --config $c --strategy $1 --no-e2e --no-cpu --no-per-config --steps 5 > $OUT/ab_${c}_$1_$2_$rep.json 2> $OUT/ab_${c}_$1_$2_$rep.err
    python -c "
import json; d=json.load(open('$OUT/ab_${c}_$1_$2_$rep.json')); print('$c $1 two=$2', d['ms_per_step'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()}, d.get('class_ms_symbolic'))" || tail -2 $OUT/ab_${c}_$1_$2_$rep.err
  done; done; done
