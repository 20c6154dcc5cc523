# parity subset + c3a/c3b benches (class breakdown)
OUT=gpurun_out/${TAG:-s3}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout ${TTIME:-1500} python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYK:+-k "$PYK"} > $OUT/t.log 2>&1; tail -5 $OUT/t.log
for c in ${CFGS:-c3a c3b}; do
for st in ${STRATS:-precise}; do
timeout 600 python bench.py --config $c --strategy $st --no-e2e --no-cpu --no-per-config --steps 3 > $OUT/b_${c}_$st.json 2> $OUT/b_${c}_$st.err
python -c "
import json; d=json.load(open('$OUT/b_${c}_$st.json')); print('$c $st', d['ms_per_step'], d['stage_ms'], d['class_ms'])" || tail -3 $OUT/b_${c}_$st.err
done; done
