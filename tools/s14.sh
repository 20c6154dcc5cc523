OUT=gpurun_out/${TAG:-s14}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYK:+-k "$PYK"} > $OUT/t.log 2>&1; tail -3 $OUT/t.log; grep FAILED $OUT/t.log | head
IFS=',' read -ra SPECS <<< "${BENCHES}"
for spec in "${SPECS[@]}"; do IFS=':' read -r t e c st <<< "$spec";
  env $e timeout 600 python bench.py --config $c --strategy $st --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/b_$t.json 2> $OUT/b_$t.err
  python -c "
import json; d=json.load(open('$OUT/b_$t.json')); print('$t', d['ms_per_step'], d['stage_ms'], {k:{c:v for c,v in x.items() if v>0.3} for k,x in d['class_ms'].items()})" || tail -3 $OUT/b_$t.err
done
