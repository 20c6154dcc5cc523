#!/bin/bash
# long-row kernels: tests + c3b / g3d27_ptap A/B (libspgemm_prev.so vs libspgemm.so)
OUT=gpurun_out/${TAG:-ablong}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "long or rank or rmat or chash or c3b or growth or arena or forced or determinism or galerkin" > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -2 $OUT/tests.log
for rep in 1 2; do for lib in libspgemm_prev.so libspgemm.so; do for c in c3b g3d27_ptap; do
  SPGEMM_LIB=$lib timeout 300 python bench.py --config $c --strategy precise --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/$c.json 2> $OUT/err
  python -c "
import json; d=json.load(open('$OUT/$c.json')); cm=d['class_ms']; print('$c $lib', d['ms_per_step'], {k: v.get('long') for k, v in cm.items()})"
done; done; done
