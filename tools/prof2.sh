#!/bin/bash
# ncu full captures of named kernels for one config: tools/prof2.sh <tag> <cfg> <strategy> <kernel-regex> [count]
TAG=$1; CFG=$2; ST=$3; KRE=$4; N=${5:-1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 0 -c $N -o $OUT/prof_${CFG}_${ST} python tools/prof_one.py $CFG $ST > $OUT/ncu_${CFG}_${ST}.log 2>&1
tail -2 $OUT/ncu_${CFG}_${ST}.log
