# K5 variant sweep on cfg5 (2^26 cells, CFG5_STEPS steps) for each variant lib
for rep in 1 2; do for v in "$@"; do
  FQNM_LIBPATH=$PWD/variants/libfqnm_$v.so CFG5_STEPS=${CFG5_STEPS:-200} timeout 300 python tools/bench_configs.py cfg5 | sed "s/^/$v /" | cut -c1-140
done; done
