#!/bin/bash
# Round evidence: full GPU tests, default bench line (+ per_config), reference arm, ncu launch
# lists (c2 precise, c3a hybrid), ncu full captures of the dominant kernels (summarised on the box).
OUT=gpurun_out/${TAG:-ev}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $OUT/gpu_tests.log 2>&1; echo TESTS_RC=$? >> $OUT/gpu_tests.log
fi
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|k_" -c 2000 --csv --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-per-config > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 2000 --csv --log-file $OUT/launches_c3a_hybrid.csv python bench.py --config c3a --strategy hybrid --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > /dev/null 2>&1
TAG=${TAG:-ev}/c2full KBASE=demangled KRE="k_bw_sym|k_bwrow<.int.3" NC3A=2 CFG1=c2 SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
TAG=${TAG:-ev}/c3a KBASE=demangled KRE="k_esc_bk|k_bk_|k_copy" NC3A=14 CFG1="c3a --strategy hybrid" SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
TAG=${TAG:-ev}/c3b KBASE=function KRE="k_long" NC3A=2 CFG1=c3b SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
tail -3 $OUT/gpu_tests.log; tail -2 $OUT/smoke.log; head -c 1500 $OUT/bench.json; echo; cat $OUT/bench_reference.json
