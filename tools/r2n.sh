#!/bin/bash
OUT=gpurun_out/${TAG:-r2n}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
bash tools/r2m.sh
bash tools/ab2.sh ${TAG:-r2n} "libspgemm.so libspgemm_ch64.so libspgemm_ch256.so libspgemm_ch1024.so" "c2" precise
