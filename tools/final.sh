#!/bin/bash
# Final evidence session: smoke, the GPU test suite, the default bench line (+ per_config),
# the reference arm, the c2 launch list, and an ncu capture of the hybrid window kernel.
OUT=gpurun_out/${TAG:-fin}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 2000 --csv --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-per-config > /dev/null 2>&1
TAG=${TAG:-fin}/c2hyb KBASE=demangled KRE="k_bw_one|k_copy_flat" NC3A=2 CFG1="c2 --strategy hybrid" SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
tail -3 $OUT/gpu_tests.log; tail -2 $OUT/smoke.log; head -c 600 $OUT/bench.json; echo
