#!/bin/bash
# hybrid with the relaxed window bound (SPGEMM_HYBRID_RELAX=1) vs strict, and precise
OUT=gpurun_out/${TAG:-r2r}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SPGEMM_HYBRID_RELAX=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "not c3a_full and not c5_rank and not c3b_full and not c4_full" > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -2 $OUT/tests.log
for c in g3d27 g3d7 g2d9 g2d5 g3d27_ptap c4b c2; do for v in "hybrid 0" "hybrid 1" "precise 0"; do set -- $v
  SPGEMM_HYBRID_RELAX=$2 timeout 300 python bench.py --config $c --strategy $1 --no-e2e --no-cpu --no-per-config --steps 5 > $OUT/$c_$1_$2.json 2> $OUT/err
  python -c "
import json; d=json.load(open('$OUT/$c_$1_$2.json')); print('$c $1 relax=$2', d['ms_per_step'])" || tail -3 $OUT/err
done; done
