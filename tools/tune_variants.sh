#!/bin/bash
# EO kernel variant sweep (libs built by paper_2604_06947_b200/_build.py with FQNM_EO_VARIANT)
B=paper_2604_06947_b200
for lib in $B/libfqnm.so $B/build/libfqnm_v5.so; do
  FQNM_LIBPATH=$PWD/$lib TUNE_V=32 TUNE_K=24 TUNE_FAM=202 python tools/tune.py eo
  FQNM_LIBPATH=$PWD/$lib TUNE_V=16 TUNE_K=16 TUNE_FAM=302 python tools/tune.py eo
done
