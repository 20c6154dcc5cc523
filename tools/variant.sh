#!/bin/bash
# Build an A/B variant of libspgemm into paper_1504_05022_b200/<name> with extra -D flags, then
# restore the default build.  usage: tools/variant.sh libspgemm_b.so "SG_PIPE_G=4 X=1"
NAME=$1; DEFS=$2
SPGEMM_DEFS="$DEFS" python -c "from paper_1504_05022_b200 import build as b; b.build(force=True)" && \
  cp paper_1504_05022_b200/libspgemm.so paper_1504_05022_b200/$NAME
python -c "from paper_1504_05022_b200 import build as b; b.build(force=True)"
