#!/bin/bash
# usage: tools/bench_some.sh <outdir> <name:args>...
OUT=$1; shift; mkdir -p $OUT
for spec in "$@"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout ${BENCH_TIMEOUT:-600} python bench.py $args > $OUT/$name.json 2> $OUT/$name.err; rc=$?
  python - $OUT/$name.json $name $rc <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("%-10s rc=%s %8.1f GFlop/s  %8.3f ms/step  hbm_frac=%.4f  stages=%s" % (sys.argv[2], sys.argv[3], d["value"], d["ms_per_step"], d["hbm"]["frac_of_peak"], d["stage_ms"]))
except Exception as e:
    print(sys.argv[2], "rc=", sys.argv[3], "no result", e)
PY
done
