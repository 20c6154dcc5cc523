#!/bin/bash
# tests touching the ESC classes + c5 at a reduced scale; optional ncu on a kernel regex
TAG=$1; KRE=$2; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${TESTK:-tier or rmat or config}" > $OUT/t.log 2>&1; tail -2 $OUT/t.log
python bench.py --config ${CFG:-c5} --scale ${SCALE:-20} --no-e2e --no-cpu --steps 3 > $OUT/b.json 2> $OUT/b.err
python -c "
import json; d=json.load(open('$OUT/b.json')); print(d['ms_per_step'], d['value'], d['stage_ms'], d['roofline']['kernel'])" || tail -3 $OUT/b.err
if [ -n "$KRE" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 2 -c 2 -o $OUT/prof python tools/prof_one.py ${CFG:-c5} precise scale=${SCALE:-20} > $OUT/ncu.log 2>&1; tail -1 $OUT/ncu.log; fi
