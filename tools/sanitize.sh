#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py
OUT=gpurun_out/${TAG:-san}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout ${STIME:-1500} compute-sanitizer --tool $tool --kernel-name regex=k_ --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_run.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $OUT/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_RUN_DONE|Error|Hazard" $OUT/$tool.log | head -8 | tee -a $OUT/summary.txt
done
