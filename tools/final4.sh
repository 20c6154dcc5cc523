#!/bin/bash
OUT=gpurun_out/${TAG:-fin4}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
timeout 2000 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/gpu_tests.log; tail -2 $OUT/smoke.log; head -c 300 $OUT/bench.json; echo
