# ncu full captures of the c3a / c3b stage-3 kernels (first pass of a 1-step bench run)
OUT=gpurun_out/${TAG:-s5}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_esc_merge|k_esc_sort|k_bk_|k_wrow|k_cta_hash|k_long" -c ${NC3A:-24} -o $OUT/c3a python bench.py --config c3a --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > $OUT/ncu_c3a.log 2>&1
tail -3 $OUT/ncu_c3a.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_long" -c 2 -o $OUT/c3b python bench.py --config c3b --steps 1 --warmup 1 --no-e2e --no-cpu --no-per-config > $OUT/ncu_c3b.log 2>&1
tail -3 $OUT/ncu_c3b.log
