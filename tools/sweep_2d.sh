# K9 variant sweep: usage bash tools/sweep_2d.sh tag1 tag2 ... (variants/libfqnm_<tag>.so)
# K9 variant sweep: default (k = 2) and k = 1 on 8192^2 EO / linear for each variant lib
B=variants
for rep in 1 2; do for v in "$@"; do
  FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so timeout 120 python tools/bench_configs.py eo2d lin2d | sed "s/^/$v k2 /"
  KERN2D=9 K2D=1 FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so timeout 120 python tools/bench_configs.py eo2d lin2d | sed "s/^/$v k1 /"
done; done
