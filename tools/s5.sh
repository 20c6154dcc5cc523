# ncu full captures of the c3a / c3b stage-3 kernels (first pass of a 1-step bench run);
# the reports are summarised on the box (raw csv + per-kernel source csv) and deleted (64 MiB cap)
OUT=gpurun_out/${TAG:-s5}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
summ() {  # $1 = report base name
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
  for k in $(ncu -i $OUT/$1.ncu-rep --page raw --csv --metrics launch__grid_size 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; i=h.index('Kernel Name')
seen=[]
for x in r[2:]:
    n=x[i].split('(')[0].split('<')[0].split('::')[-1]
    if n not in seen: seen.append(n)
print(' '.join(seen))"); do
    ncu -i $OUT/$1.ncu-rep --page source --csv --print-source cuda,sass -k regex:"$k" > $OUT/$1_src_$k.csv 2>/dev/null
    python tools/src_lines.py $OUT/$1_src_$k.csv 30 > $OUT/$1_lines_$k.txt 2>/dev/null
    rm -f $OUT/$1_src_$k.csv
  done
  python tools/profile_report.py $OUT/$1.md $OUT/$1.ncu-rep > /dev/null 2>&1
  [ -n "$KEEP" ] || rm -f $OUT/$1.ncu-rep
}
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base ${KBASE:-function} -k regex:"${KRE:-k_esc_merge|k_esc_sort|k_bk_|k_wrow|k_cta_hash|k_long}" -c ${NC3A:-24} -o $OUT/c3a python bench.py --config ${CFG1:-c3a} --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > $OUT/ncu_c3a.log 2>&1
summ c3a
if [ -z "$SKIP2" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_long" -c 2 -o $OUT/c3b python bench.py --config c3b --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > $OUT/ncu_c3b.log 2>&1
summ c3b
fi
du -sh $OUT
