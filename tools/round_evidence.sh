#!/bin/bash
# Evidence for profiles/: default bench line, ncu launch list of the same command, full
# captures of the dominant kernels (c2 precise: window-bitmap STRUCT + DENSE; c2 hybrid: FILL + copy).
OUT=${1:-gpurun_out/ev}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --strategy hybrid --no-e2e --no-cpu > $OUT/bench_hybrid.json 2> $OUT/bench_hybrid.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bw_struct2|k_bwrow" -s 9 -c 3 -o $OUT/c2_precise python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bw_struct2|k_bwrow|k_copy" -s 9 -c 3 -o $OUT/c2_hybrid python bench.py --strategy hybrid --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full_h.log 2>&1
cat $OUT/bench.json; tail -2 $OUT/bench_hybrid.json; cat $OUT/bench_reference.json
