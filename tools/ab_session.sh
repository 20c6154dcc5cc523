#!/bin/bash
OUT=gpurun_out/r2t; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
[ -n "$NOTEST" ] || timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "bw or window or stencil or config1 or strategies or c2_full or galerkin or forced or f32" > $OUT/tests.log 2>&1; echo TESTS_RC=$? >> $OUT/tests.log
tail -2 $OUT/tests.log
bash tools/ab2.sh r2t "${LIBS:-libspgemm_prev.so libspgemm.so}" "${CFGS:-c2 g3d27 g2d9}" precise
