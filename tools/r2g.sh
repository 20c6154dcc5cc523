#!/bin/bash
OUT=gpurun_out/${TAG:-r2g}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${KSEL:+-k "$KSEL"} > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -3 $OUT/tests.log
bash tools/ab2.sh ${TAG:-r2g} "${LIBS:-libspgemm_prev.so libspgemm.so}" "${CFGS:-c2}" ${ST:-hybrid}
[ -n "$BENCH" ] && timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err && python -c "
import json; d=json.load(open('$OUT/bench.json')); print(d['ms_per_step'], d['value'], d['e2e'], d['roofline']['frac'])"
