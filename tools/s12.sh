OUT=gpurun_out/${TAG:-s12}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${PYK}" > $OUT/t.log 2>&1; tail -3 $OUT/t.log
bash tools/ab2.sh ${TAG}_ab "libspgemm_a.so libspgemm.so" "${CFGS}" ${ST:-precise}
