# K8 variant sweep: libs built by _build.build(defines=[...], lib=variants/libfqnm_<tag>.so)
# usage: bash tools/sweep_3d.sh tag1 tag2 ...   (GCUPS + sha of the state, 512^3 EO / linear)
B=variants
for rep in 1 2; do for v in "$@"; do
  TAG=$v FQNM_LIBPATH=$PWD/$B/libfqnm_$v.so timeout 120 python tools/sweep_3d.py
done; done
