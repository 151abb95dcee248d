#!/bin/bash
# Kernel variant sweep: libs built by _build.build(defines=[...], lib=build/libfqnm_<tag>.so)
# usage: bash tools/variant_sweep.sh tag1 tag2 ...   (prints GCUPS + sha of the final state)
#   WHICH=eo (cfg4 slice, V=32 k=24) | lin (cfg3, V=32 k=64)
B=paper_2604_06947_b200/build
WHICH=${WHICH:-eo}
for rep in 1 2; do for v in "$@"; do
  if [ "$WHICH" = eo ]; then
    FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so TUNE_N=268435456 TUNE_V=32 TUNE_K=24 TUNE_FAM=202 timeout 120 python tools/tune.py eo | sed "s/^/$v /"
  else
    FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so TUNE_V=32 TUNE_K=${LIN_K:-64} TUNE_FAM=202 timeout 120 python tools/tune.py lin | sed "s/^/$v /"
  fi
done; done
