OUT=gpurun_out/s2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "f32" > $OUT/t.log 2>&1; tail -5 $OUT/t.log
for c in c3a c3b; do
timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/b_$c.json 2> $OUT/b_$c.err
python -c "
import json; d=json.load(open('$OUT/b_$c.json')); print('$c', d['ms_per_step'], d['stage_ms'], d['class_ms'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_c3a.csv python bench.py --config c3a --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bwrow" -s 13 -c 1 -o $OUT/dense python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-per-config > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
