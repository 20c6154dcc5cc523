#!/bin/bash
# Session: parity subset for the window class + A/B of libspgemm_old.so vs libspgemm.so.
OUT=gpurun_out/${TAG:-r2b}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${KSEL:-window or bw or stencil or forced_tier_precise or config1 or galerkin or strategies or c2_full or determinism}" > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -3 $OUT/tests.log
bash tools/ab2.sh ${TAG:-r2b} "${LIBS:-libspgemm_old.so libspgemm.so}" "${CFGS:-c2}" precise 2>&1 | tee $OUT/ab.txt
