OUT=gpurun_out/${TAG:-s6}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout ${TTIME:-1500} python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYK:+-k "$PYK"} > $OUT/t.log 2>&1; tail -5 $OUT/t.log
b() { # tag env config strategy
  env $2 timeout 600 python bench.py --config $3 --strategy $4 --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/b_$1.json 2> $OUT/b_$1.err
  python -c "
import json; d=json.load(open('$OUT/b_$1.json')); print('$1', d['ms_per_step'], d['stage_ms'], d['class_ms'], d.get('class_ms_symbolic'))" || tail -3 $OUT/b_$1.err
}
# BENCHES="tag:ENV=val:config:strategy,..."
IFS=',' read -ra SPECS <<< "${BENCHES:-c3a_new:X=1:c3a:precise}"
for spec in "${SPECS[@]}"; do IFS=':' read -r t e c st <<< "$spec"; b $t $e $c $st; done
