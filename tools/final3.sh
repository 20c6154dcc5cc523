#!/bin/bash
# Final bench line (+ per_config), c2 launch list, ncu capture of the c2 precise window kernels.
OUT=gpurun_out/${TAG:-fin3}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
timeout 2000 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 2000 --csv --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-per-config > /dev/null 2>&1
TAG=${TAG:-fin3}/c2full KBASE=demangled KRE="k_bw_sym|k_bwrow<.int.3" NC3A=2 CFG1=c2 SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
tail -2 $OUT/smoke.log; head -c 300 $OUT/bench.json; echo
