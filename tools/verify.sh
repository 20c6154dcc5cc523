#!/bin/bash
# Verification session: smoke, the GPU test suite, the default bench line.
OUT=gpurun_out/${TAG:-verify}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 -x > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
fi
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/gpu_tests.log; tail -2 $OUT/smoke.log; head -c 3000 $OUT/bench.json
