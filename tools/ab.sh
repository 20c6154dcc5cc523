#!/bin/bash
# A/B timing in one GPU session: libspgemm_a.so (A) vs libspgemm.so (B), alternating.
# usage: tools/ab.sh <bench args...>
for i in 1 2; do
  for lib in libspgemm_a.so libspgemm.so; do
    SPGEMM_LIB=$lib python bench.py --no-e2e --no-cpu "$@" 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$lib', d['ms_per_step'], {k: [round(x,2) for x in v] for k,v in d['stage_ms'].items()})"
  done
done
