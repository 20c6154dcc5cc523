#!/bin/bash
OUT=gpurun_out/${TAG:-r2s}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
tail -3 $OUT/gpu_tests.log
for c in c3a g3d27_ptap g2d9; do for st in hybrid; do
  timeout 300 python bench.py --config $c --strategy $st --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/$c_$st.json 2> $OUT/err
  python -c "
import json; d=json.load(open('$OUT/$c_$st.json')); print('$c $st', d['ms_per_step'], d.get('class_ms'))" | cut -c1-400
done; done
