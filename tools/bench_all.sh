#!/bin/bash
# All BASELINE configs through bench.py (1 GPU).  usage: tools/bench_all.sh <outdir>
OUT=${1:-gpurun_out/all}; mkdir -p $OUT
run() { name=$1; shift; timeout 1200 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; tail -c 600 $OUT/$name.json; echo; }
run c2_precise --config c2 --strategy precise
run c2_hybrid --config c2 --strategy hybrid --no-cpu --no-e2e
run c1 --config c1 --no-e2e --no-cpu
run c4a --config c4a --no-e2e --no-cpu
run c4b --config c4b --no-e2e --no-cpu
run c3b --config c3b --no-e2e --no-cpu
run c5_s19 --config c5 --scale 19 --no-e2e --no-cpu
run c3a --config c3a --no-e2e --no-cpu --steps 5
