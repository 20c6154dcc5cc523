#!/bin/bash
# VMM arena cache: tests of the long-row paths, host timeline and bench of c3b hybrid, old vs new.
OUT=gpurun_out/${TAG:-r2m}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${KSEL:-long or arena or growth or strategies or rmat or c3b}" > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -3 $OUT/tests.log
for lib in libspgemm_prev.so libspgemm.so; do
  echo "== $lib"; SPGEMM_LIB=$lib timeout 600 python tools/steptime.py c3b hybrid 2>&1 | tail -3
done
bash tools/ab2.sh ${TAG:-r2m} "libspgemm_prev.so libspgemm.so" "c3b" hybrid
