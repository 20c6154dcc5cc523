#!/bin/bash
# Final bench line (+ per_config, both strategies), reference arm, ncu capture of k_bw_one.
OUT=gpurun_out/${TAG:-fin2}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo SMOKE_RC=$? >> $OUT/smoke.log
timeout 2000 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
TAG=${TAG:-fin2}/c2hyb KBASE=demangled KRE="k_bw_one|k_copy_flat" NC3A=2 CFG1="c2 --strategy hybrid" SKIP2=1 bash tools/s5.sh > /dev/null 2>&1
tail -2 $OUT/smoke.log; head -c 400 $OUT/bench.json; echo
